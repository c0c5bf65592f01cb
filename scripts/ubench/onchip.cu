// Microbenchmarks for an on-chip-resident shard kernel (one CTA per SM, 256 threads):
//  (1) TMEM as a per-thread store of cost values: tcgen05.ld.32x32b.x16 -> FFMA + MUFU.EX2 + FADD; ex2/clk/SM
//      for the TMEM-only, smem-only and mixed (half/half) loops;
//  (2) a device-wide column-sum reduction through 64-bit integer atomics (red.global.add.u64, cumulative
//      per-parity sums, one cumulative arrival counter per column group): iteration time of
//      {W reds per CTA -> arrive -> poll -> read W sums} for W = 1024 / 512 / 256 columns per CTA.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

#define TLD16(taddr, r)                                                                                        \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}," \
               " [%16];"                                                                                       \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), \
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),       \
                 "=r"(r[15])                                                                                   \
               : "r"(taddr))
#define TST16(taddr, r)                                                                                         \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
               "%16};" ::"r"(taddr),                                                                            \
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),  \
               "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]))

// MODE 0: TMEM only (256 words per thread), 1: smem only (thread-private 1 KB column), 2: both (TMEM 1 KB then
// smem 1 KB per thread: 2 KB of values per thread, 512 KB per CTA... smem part capped at 192 B/thread*...)
template <int MODE>
__global__ void __launch_bounds__(256, 1) k_tmem(float* out, int iters, int smem_words) {
  extern __shared__ __align__(16) float sm[];
  __shared__ unsigned tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned ta = tbase + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)((warp >> 2) * 256);
  for (int c = 0; c < 256; c += 16) {
    unsigned r[16];
    for (int q = 0; q < 16; ++q) r[q] = __float_as_uint(0.001f * ((c + q + threadIdx.x) & 31));
    TST16(ta + c, r);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  for (int i = threadIdx.x; i < smem_words * 256; i += 256) sm[i] = 0.002f * (i & 15);
  __syncthreads();
  const float c2 = 1.7f, g = 0.3f;
  float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
  const float4* s4 = reinterpret_cast<const float4*>(sm);
  for (int it = 0; it < iters; ++it) {
    if (MODE != 1) {
#pragma unroll 1
      for (int c = 0; c < 256; c += 32) {
        unsigned a[16], b[16];
        TLD16(ta + c, a);
        TLD16(ta + c + 16, b);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float e[32];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          e[q] = ex2(fmaf(-__uint_as_float(a[q]), c2, g));
          e[16 + q] = ex2(fmaf(-__uint_as_float(b[q]), c2, g));
        }
#pragma unroll
        for (int q = 0; q < 32; q += 4) {
          acc0 += e[q];
          acc1 += e[q + 1];
          acc2 += e[q + 2];
          acc3 += e[q + 3];
        }
      }
    }
    if (MODE != 0) {
      // thread-private values interleaved across threads: word (k, v) of thread t at float4 index k*256 + t
#pragma unroll 1
      for (int k = 0; k < smem_words / 4; k += 4) {
        float4 c[4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) c[kk] = s4[(size_t)(k + kk) * 256 + threadIdx.x];
        float e[16];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          e[4 * kk] = ex2(fmaf(-c[kk].x, c2, g));
          e[4 * kk + 1] = ex2(fmaf(-c[kk].y, c2, g));
          e[4 * kk + 2] = ex2(fmaf(-c[kk].z, c2, g));
          e[4 * kk + 3] = ex2(fmaf(-c[kk].w, c2, g));
        }
#pragma unroll
        for (int q = 0; q < 16; q += 4) {
          acc0 += e[q];
          acc1 += e[q + 1];
          acc2 += e[q + 2];
          acc3 += e[q + 3];
        }
      }
    }
  }
  out[blockIdx.x * 256 + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

// ---- device-wide reduction through u64 atomics
__global__ void __launch_bounds__(256, 1) k_atomred(unsigned long long* sums, unsigned* cnt, int iters, int W,
                                                     int h, long long* out_cycles) {
  extern __shared__ __align__(16) float sm[];   // only to force one CTA per SM
  const int grp = blockIdx.x % h;               // column group of this CTA
  const int G = gridDim.x / h;                  // CTAs per group (grid is a multiple of h)
  const int m = W * h;
  unsigned long long prev[4];
  // baselines: grid barrier first
  cooperative_groups::this_grid().sync();
  for (int q = 0; q < 4; ++q) {
    const int j = threadIdx.x + q * 256;
    prev[q] = j < W ? *(volatile unsigned long long*)&sums[(size_t)grp * W + j] : 0ull;
  }
  const unsigned c0 = *(volatile unsigned*)&cnt[grp];
  cooperative_groups::this_grid().sync();
  unsigned long long chk = 0;
  const long long t0 = clock64();
  for (int t = 0; t < iters; ++t) {
    unsigned long long* S = sums + (size_t)(t & 1) * m + (size_t)grp * W;
    for (int q = 0; q < 4; ++q) {
      const int j = threadIdx.x + q * 256;
      if (j < W) {
        const unsigned long long v = 1000ull + blockIdx.x + t;
        asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(S + j), "l"(v) : "memory");
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cnt + grp) : "memory");
      const unsigned want = c0 + (unsigned)G * (unsigned)(t + 1);
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt + grp) : "memory");
      } while ((int)(v - want) < 0);
    }
    __syncthreads();
    for (int q = 0; q < 4; ++q) {
      const int j = threadIdx.x + q * 256;
      if (j < W) {
        unsigned long long v;
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(S + j) : "memory");
        chk += v - ((t & 1) ? 0 : 0);
      }
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) out_cycles[blockIdx.x] = t1 - t0;
  if (chk == 42) out_cycles[0] = 0;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, sms * 256 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // (1) TMEM
  for (int mode = 0; mode < 3; ++mode) {
    const int sw = mode == 0 ? 4 : 192;   // smem words per thread (192 B... x4 B = 768 B per thread)
    const size_t smem = (size_t)sw * 256 * 4;
    void* fn = mode == 0 ? (void*)k_tmem<0> : mode == 1 ? (void*)k_tmem<1> : (void*)k_tmem<2>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int iters = 2000;
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k_tmem<0><<<sms, 256, smem>>>(out, iters, sw);
      if (mode == 1) k_tmem<1><<<sms, 256, smem>>>(out, iters, sw);
      if (mode == 2) k_tmem<2><<<sms, 256, smem>>>(out, iters, sw);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double per_thread = (mode != 1 ? 256.0 : 0.0) + (mode != 0 ? (double)sw : 0.0);
    const double ex = (double)sms * 256 * per_thread * iters;
    printf("tmem mode %d (%s): %.2f ex2 per SM per clk (@ %d MHz nominal)  %s\n", mode,
           mode == 0 ? "TMEM" : mode == 1 ? "smem" : "TMEM+smem", ex / (best * 1e-3) / sms / (clk * 1e3),
           clk / 1000, cudaGetErrorString(cudaGetLastError()));
  }
  // (2) atomics
  unsigned long long* sums;
  unsigned* cnt;
  long long* cyc;
  cudaMalloc(&sums, 2 * 1024 * 8);
  cudaMalloc(&cnt, 64 * 4);
  cudaMalloc(&cyc, sms * 8);
  cudaMemset(sums, 0, 2 * 1024 * 8);
  cudaMemset(cnt, 0, 64 * 4);
  cudaFuncSetAttribute(k_atomred, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int cfg[][2] = {{1024, 1}, {512, 2}, {256, 4}, {128, 4}};
  for (auto& c : cfg) {
    int W = c[0], h = c[1];
    int grid = sms / h * h;
    int iters = 2000;
    void* args[] = {&sums, &cnt, &iters, &W, &h, &cyc};
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((void*)k_atomred, grid, 256, args, 200 * 1024, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("atomred W=%d h=%d grid=%d: %.3f us per iteration (%d reds per iteration)  %s\n", W, h, grid,
           best * 1e3 / iters, grid * W, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
