// Device helpers shared by the sm_100a kernels of libcyclicot (no torch, no host logic).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/cyclicot.h"

#define COT_LOG2E 1.4426950408889634
#define COT_LN2 0.6931471805599453

namespace cot {

// ------------------------------------------------------------------------------------- math
// MUFU.EX2 with flush-to-zero: 2^x, max rel. error ~2 ulp; x <= 0 in every use here.
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x = 2^k * 2^f with k = round(x) an integer and 2^f (|f| <= 1/2) in fp64 (the 1.5 * 2^52 rounding trick,
// valid for |x| < 2^31). Explicitly rounded operations: the compiler must not contract them into FMAs
// differently at different call sites (the split of a z value has to be bitwise the same wherever it is taken,
// or launches that continue each other would not reproduce a single launch).
__device__ __forceinline__ double split_pow2_fp64(double x, int& k) {
  const double big = __dadd_rn(x, 6755399441055744.0);   // 1.5 * 2^52: round to an integer in the low word
  k = __double2loint(big);
  return exp2(__dsub_rn(x, __dsub_rn(big, 6755399441055744.0)));
}
// The split of a potential z (natural units): z log2e = k + f.
__device__ __forceinline__ double split_z(double z, int& k) { return split_pow2_fp64(__dmul_rn(z, COT_LOG2E), k); }
// f * 2^e, exactly, for f in [2^-22, 2^23) (the k-sums s'_ij lie in [0.7, 1.42 n]) and e clamped to
// [-1000, 1000]: terms below 2^-1000 come out ~1e-301 (negligible); callers whose exponents can exceed 1000
// check the sums' range. Integer operations only.
__device__ __forceinline__ double ldexp_pos(float f, int e) {
  const unsigned b = __float_as_uint(f);
  e = min(max(e, -1000), 1000);
  return __hiloint2double((int)((b >> 3) + ((unsigned)(e + 896) << 20)), (int)(b << 29));
}

// 1/r for a positive normal fp64 r without the MUFU pipe (kernels whose k-sum warps keep MUFU.EX2 saturated
// would otherwise queue the epilogue's MUFU.RCP behind them): exponent-negation estimate (relative error
// <= 5.1%) and four Newton steps (quadratic: 2.6e-3, 6.5e-6, 4.2e-11, rounding level; checked on 4e4 samples
// over [1e-280, 1e280]).
__device__ __forceinline__ double rcp_nomufu(double r) {
  double y = __hiloint2double(0x7FDE6239 - __double2hiint(r), 0);
#pragma unroll
  for (int s = 0; s < 4; ++s) y = fma(y, fma(-r, y, 1.0), y);
  return y;
}

// log(x) for a positive normal fp64 x without the MUFU pipe (CUDA's log issues one MUFU.RCP64H, which queues
// behind the k-sum warps' MUFU.EX2 on the per-iteration critical path): x = m 2^e with m in [1/sqrt2, sqrt2),
// log m = 2 atanh(s), s = (m - 1)/(m + 1), |s| <= 0.1716, odd series to s^25 (truncation < 1e-20); error
// <= 5e-16 (relative, or absolute near x = 1) on 4e4 samples over [1e-30, 1e3].
__device__ __forceinline__ double log_nomufu(double x) {
  const int hi = __double2hiint(x);
  int e = (hi >> 20) - 1023;
  double m = __hiloint2double((hi & 0x000FFFFF) | 0x3FF00000, __double2loint(x));
  if (m > 1.4142135623730951) {
    m *= 0.5;
    e += 1;
  }
  const double s = (m - 1.0) * rcp_nomufu(m + 1.0), s2 = s * s;
  double p = 1.0 / 25;
#pragma unroll
  for (int k = 23; k >= 1; k -= 2) p = fma(p, s2, 1.0 / k);
  return fma((double)e, COT_LN2, 2.0 * s * p);
}

__device__ __forceinline__ bool finite_f(float x) { return fabsf(x) <= 3.402823466e38f; }
__device__ __forceinline__ bool finite_f(double x) { return fabs(x) <= 1.7976931348623157e308; }

// --------------------------------------------------------------------------------- reductions
template <typename V>
__device__ __forceinline__ V warp_sum(V v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename V>
__device__ __forceinline__ V warp_max(V v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide reductions over the first NW warps (NW = blockDim/32), fixed order => deterministic.
// `scratch` must hold NW doubles; it is reused, so consecutive calls are separated by a barrier.
template <int NW>
__device__ __forceinline__ double block_sum(double v, double* scratch, int bar_id, int nthreads) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) scratch[wid] = v;
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthreads));
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < NW; ++w) t += scratch[w];
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthreads));
  return t;
}
template <int NW>
__device__ __forceinline__ double block_max(double v, double* scratch, int bar_id, int nthreads) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_max(v);
  if (lane == 0) scratch[wid] = v;
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthreads));
  double t = scratch[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) t = fmax(t, scratch[w]);
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthreads));
  return t;
}

// ---------------------------------------------------------------------- mbarrier + bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk async copy global -> shared (TMA engine; SASS UBLKCP), completion on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// streaming stores (evict-first) for write-once outputs
__device__ __forceinline__ void st_cs(float4* p, float4 v) { __stcs(p, v); }
__device__ __forceinline__ void st_cs(float* p, float v) { __stcs(p, v); }
__device__ __forceinline__ void st_cs(double* p, double v) { __stcs(p, v); }
__device__ __forceinline__ void st_cs(double2* p, double2 v) { __stcs(p, v); }

}  // namespace cot
