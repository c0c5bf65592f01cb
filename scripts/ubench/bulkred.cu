// Microbenchmark: device-wide column-sum reduction with TMA bulk reductions (cp.reduce.async.bulk .add.u64) whose
// 64-bit sums carry their contribution count in the top byte (k_iter_res.cu's device-wide step), 148 CTAs x W
// columns, K replicas of the sum buffer (CTA c adds into replica c % K; readers poll all K) to spread the same-address
// atomic traffic. Prints us per iteration (reduce -> every CTA holds its W sums).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p, int sys) {
  unsigned long long v;
  if (sys) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__global__ void __launch_bounds__(256, 1) k_bulkred(unsigned long long* sums, int W, int K, int iters, int sys,
                                                    unsigned long long* out, int sent, int mode) {
  extern __shared__ __align__(128) unsigned long long cb[];
  const int c = blockIdx.x, G = gridDim.x;
  const int rep = c % K;
  const unsigned want = (unsigned)(G / K + (rep < G % K ? 1 : 0));
  unsigned long long acc = 0;
  const int zslice = (W * K + G - 1) / G;
  for (int t = 0; t < iters; ++t) {
    const int sl = t % 3, slp = (t + 2) % 3;
    if (mode == 1) {   // individual coalesced reductions, count in the top byte
      if (threadIdx.x == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");
      __syncthreads();
      for (int j = threadIdx.x; j < W; j += 256)
        asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(sums + ((size_t)sl * K + rep) * W + j),
                     "l"((1ull << 56) | (unsigned long long)(c + j + t))
                     : "memory");
    }
    if (mode == 0) for (int j = threadIdx.x; j < W; j += 256) cb[j] = (1ull << 56) | (unsigned long long)(c + j + t);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0 && mode == 0) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      asm volatile("fence.proxy.async.global;" ::: "memory");
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u64 [%0], [%1], %2;" ::"l"(
                       sums + ((size_t)sl * K + rep) * W),
                   "r"(smem_u32(cb)), "r"((unsigned)(W * 8))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    // poll the thread's columns in every replica (sentinel mode: thread 0 first waits for the region's last
    // column, then every thread reads -- and verifies -- its own)
    if (sent) {
      if (threadIdx.x == 0)
        for (int k = 0; k < K; ++k) {
          const unsigned wk = (unsigned)(G / K + (k < G % K ? 1 : 0));
          unsigned long long v;
          do {
            v = ld_acq(sums + ((size_t)sl * K + k) * W + W - 1, sys);
            if ((unsigned)(v >> 56) == wk) break;
            if (sent > 1) __nanosleep(sent);
          } while (true);
        }
      __syncthreads();
    }
    for (int j = threadIdx.x; j < W; j += 256) {
      unsigned long long s = 0;
      for (int k = 0; k < K; ++k) {
        const unsigned wk = (unsigned)(G / K + (k < G % K ? 1 : 0));
        unsigned long long v;
        do { v = ld_acq(sums + ((size_t)sl * K + k) * W + j, sys); } while ((unsigned)(v >> 56) != wk);
        s += v & ((1ull << 56) - 1);
      }
      acc += s;
    }
    // zero this CTA's slice of the previous slot
    for (int z = threadIdx.x; z < zslice; z += 256) {
      const int idx = c * zslice + z;
      if (idx < W * K) sums[(size_t)slp * K * W + idx] = 0ull;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  out[c * 256 + threadIdx.x] = acc + want;
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *sums, *out;
  cudaMalloc(&sums, 3 * 16 * 1024 * 8);
  cudaMalloc(&out, sms * 256 * 8);
  cudaFuncSetAttribute(k_bulkred, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode : {0, 1})
  for (int sent : {0, 1})
  for (int sys = 0; sys < 1; ++sys)
    for (int W : {1024, 512, 256})
      for (int K : {1}) {
        cudaMemset(sums, 0, 3 * 16 * 1024 * 8);
        int iters = 1000;
        void* args[] = {&sums, &W, &K, &iters, &sys, &out, &sent, &mode};
        float best = 1e9;
        for (int r = 0; r < 3; ++r) {
          cudaMemset(sums, 0, 3 * 16 * 1024 * 8);
          cudaEventRecord(e0);
          cudaLaunchCooperativeKernel((void*)k_bulkred, sms, 256, args, 200 * 1024, 0);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) best = ms;
        }
        printf("%s sent=%d %s W=%4d K=%d: %.3f us/iter  %s\n", mode ? "red " : "bulk", sent, sys ? "acq.sys" : "relaxed", W, K, best * 1e3 / iters,
               cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
