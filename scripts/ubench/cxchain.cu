// Microbenchmark: the per-iteration exchange chain of a cluster-based persistent Sinkhorn kernel, without the
// row work. K clusters of S CTAs (1 CTA per SM, `smem` bytes of dynamic shared memory to get the real
// occupancy). Per iteration:
//   1. every CTA pushes its m-length partial to the column-slice owners of its cluster (DSMEM st.async with
//      mbarrier complete_tx on the owner),
//   2. each owner sums the S partials of its slice (fixed order), posts them as LL lines (L2), polls the K
//      clusters' lines of the slice and sums them in cluster order,
//   3. computes z for the slice (a log) and pushes it to every CTA of its cluster (st.async + complete_tx).
// Prints us/iteration. Usage: cxchain S K [m] [iters] [smem]
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_f64x2(uint32_t raddr, double a, double b, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "d"(a), "d"(b), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double a, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(raddr), "d"(a),
               "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void bulk_s2cl(uint32_t rdst, const void* src, uint32_t bytes, uint32_t rbar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   rdst),
               "r"(su32(src)), "r"(bytes), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void arrive_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cl(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
          su32(b)),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void st_line(uint4* p, uint4 v) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 ld_line(const uint4* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ uint4 pack(double v, unsigned g) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return make_uint4((unsigned)b, g, (unsigned)(b >> 32), g);
}
__device__ __forceinline__ double unpack(uint4 l) {
  return __longlong_as_double((long long)(((unsigned long long)l.z << 32) | l.x));
}

struct P {
  int S, K, m, iters, mode;
  uint4* lines;   // [2][K][m]
  double* out;
  unsigned long long* t;
};

__global__ void __launch_bounds__(256, 1) k_chain(P p) {
  extern __shared__ __align__(16) unsigned char sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int S = p.S, K = p.K, m = p.m;
  const int crank = (int)cl.block_rank();
  const int kc = blockIdx.x / S;   // cluster index
  const int cw = m / S;            // columns per slice
  double* pbuf = reinterpret_cast<double*>(sm);   // [S][cw] partials pushed by the cluster's CTAs
  double* zbuf = pbuf + (size_t)S * cw;           // [m] z
  double* stage = zbuf + m;                       // [m] staging for bulk copies
  double* zst = stage + m;                         // [cw] z of the own slice (bulk mode)
  uint64_t* bars = reinterpret_cast<uint64_t*>(zst + cw);   // [0] P, [1] Z
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int j = threadIdx.x; j < m; j += blockDim.x) zbuf[j] = 0.0;
  cl.sync();
  const int t4 = threadIdx.x;   // columns 4*t4 .. 4*t4+3 (m = 1024, 256 threads)
  double part[4];
  unsigned long long t0 = 0, ph[4] = {0, 0, 0, 0};
  for (int it = 0; it < p.iters; ++it) {
    if (it == 10) t0 = clock64();
    const uint32_t par = it & 1;
    if (threadIdx.x == 0) {
      arrive_expect(&bars[0], (uint32_t)(S * cw * 8));
      arrive_expect(&bars[1], (uint32_t)(m * 8));
    }
    // "epilogue": a partial that depends on z
    for (int v = 0; v < 4; ++v) {
      const int j = 4 * t4 + v;
      part[v] = j < m ? 1.0 / (1.0 + fabs(zbuf[j])) + 1e-3 * (crank + 1) : 0.0;
    }
    // 1. push to the slice owner (DSMEM)
    unsigned long long ta = clock64();
    if (p.mode == 0) {
      if (4 * t4 < m) {
        const int j = 4 * t4, o = j / cw, jj = j - o * cw;
        const uint32_t dst = mapa(su32(pbuf + (size_t)crank * cw + jj), o);
        const uint32_t rb = mapa(su32(&bars[0]), o);
        st_async_f64x2(dst, part[0], part[1], rb);
        st_async_f64x2(dst + 16, part[2], part[3], rb);
      }
    } else {   // stage locally, then one bulk copy per owner
      for (int v = 0; v < 4; ++v)
        if (4 * t4 + v < m) stage[4 * t4 + v] = part[v];
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x < S) {
        const int o = threadIdx.x;
        bulk_s2cl(mapa(su32(pbuf + (size_t)crank * cw), o), stage + (size_t)o * cw, cw * 8, mapa(su32(&bars[0]), o));
      }
    }
    unsigned long long tb = clock64();
    mbar_wait_cl(&bars[0], par);
    unsigned long long tc = clock64();
    const unsigned g = it + 1;
    uint4* lp = p.lines + (size_t)par * K * m;
    const int c = threadIdx.x;
    double cs = 0.0;
    if (c < cw) {
      double acc = 0.0;
      for (int s = 0; s < S; ++s) acc += pbuf[(size_t)s * cw + c];
      st_line(lp + (size_t)kc * m + crank * cw + c, pack(acc, g));
      for (int k0 = 0; k0 < K; k0 += 8) {
        uint4 l[8];
        unsigned todo = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (k0 + q < K) {
            l[q] = ld_line(lp + (size_t)(k0 + q) * m + crank * cw + c);
            if (!(l[q].y == g && l[q].w == g)) todo |= 1u << q;
          }
        while (todo) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (todo & (1u << q)) {
              l[q] = ld_line(lp + (size_t)(k0 + q) * m + crank * cw + c);
              if (l[q].y == g && l[q].w == g) todo &= ~(1u << q);
            }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (k0 + q < K) cs += unpack(l[q]);
      }
      const double z = log(cs);
      // 3. z of the slice to every CTA of the cluster
      if (p.mode == 0)
        for (int r = 0; r < S; ++r) st_async_f64(mapa(su32(zbuf + crank * cw + c), r), z, mapa(su32(&bars[1]), r));
      else
        zst[c] = z;
    }
    if (p.mode != 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x < S)
        bulk_s2cl(mapa(su32(zbuf + crank * cw), threadIdx.x), zst, cw * 8, mapa(su32(&bars[1]), threadIdx.x));
    }
    unsigned long long tz = clock64();
    mbar_wait_cl(&bars[1], par);
    if (it >= 10) {
      ph[0] += tb - ta;
      ph[1] += tc - tb;
      ph[2] += tz - tc;
      ph[3] += clock64() - tz;
    }
  }
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) {
    p.t[blockIdx.x * 5] = t1 - t0;
    for (int q = 0; q < 4; ++q) p.t[blockIdx.x * 5 + 1 + q] = ph[q];
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) p.out[0] = zbuf[0];
  cl.sync();
}

int main(int argc, char** argv) {
  const int S = argc > 1 ? atoi(argv[1]) : 16, K = argc > 2 ? atoi(argv[2]) : 8;
  const int m = argc > 3 ? atoi(argv[3]) : 1024, iters = argc > 4 ? atoi(argv[4]) : 2000;
  const int smem = argc > 5 ? atoi(argv[5]) : 190 * 1024;
  const int mode = argc > 6 ? atoi(argv[6]) : 0;
  P p;
  p.mode = mode;
  p.S = S;
  p.K = K;
  p.m = m;
  p.iters = iters;
  cudaMalloc(&p.lines, (size_t)2 * K * m * 16);
  cudaMemset(p.lines, 0, (size_t)2 * K * m * 16);
  cudaMalloc(&p.out, 8);
  cudaMalloc(&p.t, 8 * 5 * S * K);
  cudaFuncSetAttribute(k_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_chain, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(S * K);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = S;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int maxc = -1;
  cudaOccupancyMaxActiveClusters(&maxc, (void*)k_chain, &cfg);
  if (maxc < K) {
    printf("S=%d K=%d: only %d clusters co-resident\n", S, K, maxc);
    return 1;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, k_chain, p);   // warm-up
  cudaMemset(p.lines, 0, (size_t)2 * K * m * 16);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k_chain, p);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  static unsigned long long ht[5 * 4096];
  cudaMemcpy(ht, p.t, 8 * 5 * S * K, cudaMemcpyDeviceToHost);
  double mx = 0, ph[4] = {0, 0, 0, 0};
  for (int i = 0; i < S * K; ++i) {
    mx = ht[5 * i] > mx ? ht[5 * i] : mx;
    for (int q = 0; q < 4; ++q) ph[q] += (double)ht[5 * i + 1 + q] / (S * K) / (iters - 10);
  }
  printf("S=%2d K=%2d m=%d mode=%d (max %d clusters): %.3f us/iter (event), %.0f cycles/iter (CTA max); phases "
         "(mean cycles): epi+push %.0f, wait P %.0f, sum+L2+log+zpush %.0f, wait Z %.0f %s\n",
         S, K, m, mode, maxc, ms * 1e3 / iters, mx / (iters - 10), ph[0], ph[1], ph[2], ph[3], cudaGetErrorString(e));
  return 0;
}
