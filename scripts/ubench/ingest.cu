// Microbenchmark: per-SM ingest bandwidth into the SMs (one CTA per SM, every SM streams its own region), from L2
// (small total, re-read) or HBM (large total), by
//   mode 0: 1-D TMA bulk copies (cp.async.bulk, 4 KB each, 8 per 32 KB slot) into a 6-slot shared-memory ring,
//           one issuing lane, consumer warps only acknowledge the slots (as the persistent kernel's ring);
//   mode 1: LDG.128 (ld.global.nc.v4) into registers, 8 loads in flight per thread, 512 threads;
//   mode 2: both at once, half of the region each.
// Prints bytes per clock per SM and TB/s. Usage: ingest
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void waitp(uint64_t* b, uint32_t par) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                   su32(b)),
               "r"(par)
               : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ float4 ldg_nc(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}

constexpr int NS = 6, SLOT = 32768, CHUNK = 4096;

__global__ void __launch_bounds__(512, 1) k_ingest(const char* __restrict__ src, size_t per_cta, int mode, int reps,
                                                   float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * SLOT);
  uint64_t* empty = full + NS;
  const char* base = src + (size_t)blockIdx.x * per_cta;
  const size_t tma_bytes = (mode == 0 || mode >= 3) ? per_cta : mode == 1 ? 0 : per_cta / 2;
  const char* lbase = base + tma_bytes;
  const size_t ldg_bytes = per_cta - tma_bytes;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // roles: mode 0: warp 0 lane 0 produces, warps 1..15 consume; mode 1: all 16 warps LDG;
  //        mode 2: warps 0..7 LDG, warp 8 lane 0 produces, warps 9..15 consume
  const int prod_warp = mode == 2 ? 8 : 0;
  const bool tma_role = mode != 1 && warp >= prod_warp;
  const int ncons = mode == 2 ? 7 : 15;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], ncons);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  float acc = 0.f;
  const size_t nslots = tma_bytes / SLOT;
  if (tma_role) {
    if (warp == prod_warp) {
      if (lane == 0) {
        size_t it = 0;
        for (int r = 0; r < reps; ++r)
          for (size_t si = 0; si < nslots; ++si, ++it) {
            const int s = (int)(it % NS);
            const uint32_t ph = (uint32_t)(it / NS) & 1u;
            waitp(&empty[s], ph ^ 1u);
            expect(&full[s], SLOT);
            if (mode == 3 || mode == 4) {   // the persistent kernel's pattern: 4 KB rows 512 KB apart, evict_last
              uint64_t pol;
              asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
              const size_t nchunk = per_cta / CHUNK;   // chunk q of this CTA lives at (q * gridDim.x + blockIdx.x)
              for (int c = 0; c < SLOT / CHUNK; ++c) {
                const size_t q = (si * (SLOT / CHUNK) + c) % nchunk;
                const char* g = src + (q * gridDim.x + blockIdx.x) * (size_t)CHUNK;
                if (mode == 3)
                  bulk(sm + s * SLOT + c * CHUNK, g, CHUNK, &full[s]);
                else
                  bulk_hint(sm + s * SLOT + c * CHUNK, g, CHUNK, &full[s], pol);
              }
            } else {
              for (int c = 0; c < SLOT / CHUNK; ++c)
                bulk(sm + s * SLOT + c * CHUNK, base + si * SLOT + c * CHUNK, CHUNK, &full[s]);
            }
          }
      }
    } else {
      size_t it = 0;
      for (int r = 0; r < reps; ++r)
        for (size_t si = 0; si < nslots; ++si, ++it) {
          const int s = (int)(it % NS);
          const uint32_t ph = (uint32_t)(it / NS) & 1u;
          waitp(&full[s], ph);
          acc += reinterpret_cast<const float*>(sm + s * SLOT)[threadIdx.x & 255];
          __syncwarp();
          if (lane == 0) arrive(&empty[s]);
        }
    }
  } else {
    const int nthr = mode == 1 ? 512 : 256;
    const float4* p = reinterpret_cast<const float4*>(lbase);
    const size_t nv = ldg_bytes / 16;
    for (int r = 0; r < reps; ++r) {
      size_t i = threadIdx.x;
      for (; i + 7 * nthr < nv; i += 8 * nthr) {
        float4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = ldg_nc(p + i + (size_t)k * nthr);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += v[k].x + v[k].w;
      }
      for (; i < nv; i += nthr) acc += ldg_nc(p + i).y;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const size_t smem = NS * SLOT + 2 * NS * 8;
  cudaFuncSetAttribute(k_ingest, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  float* out;
  cudaMalloc(&out, (size_t)sms * 512 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Case { const char* name; size_t per_cta; int reps; };
  const Case cases[] = {{"L2 (192 KB/SM, x64)", 192 * 1024, 64}, {"HBM (16 MB/SM)", 16u << 20, 1}};
  for (const Case& c : cases) {
    char* src;
    cudaMalloc(&src, c.per_cta * sms);
    cudaMemset(src, 1, c.per_cta * sms);
    for (int mode = 0; mode < 5; ++mode) {
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        k_ingest<<<sms, 512, smem>>>(src, c.per_cta, mode, c.reps, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
      }
      const double bytes = (double)c.per_cta * sms * c.reps;
      printf("%-22s mode %d (%s): %.2f TB/s, %.1f B/clk/SM at %d MHz  %s\n", c.name, mode,
             mode == 0 ? "TMA" : mode == 1 ? "LDG" : mode == 2 ? "TMA+LDG" : mode == 3 ? "TMA strided" : "TMA strided evict_last", bytes / (best * 1e-3) / 1e12,
             bytes / (best * 1e-3) / sms / (clk * 1e3), clk / 1000, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(src);
  }
  return 0;
}
