// Microbenchmark: cluster signalling latency on this GPU -- a ping-pong between CTA 0 and CTA r of one cluster
// (i) through remote mbarrier arrivals (mbarrier.arrive.release.cluster on the peer's barrier, try_wait.acquire
// .cluster on the own), (ii) through DSMEM LL stores polled locally, and (iii) barrier.cluster round trips.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void __cluster_dims__(8, 1, 1) k_pp(int rounds, int peer, long long* out) {
  __shared__ __align__(8) unsigned long long bar;
  __shared__ volatile unsigned flag;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    flag = 0;
  }
  cl.sync();
  const unsigned other = rank == 0 ? peer : 0;
  const bool active = threadIdx.x == 0 && (rank == 0 || rank == (unsigned)peer);
  long long t0 = clock64();
  if (active) {   // (i) mbarrier ping-pong
    unsigned remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(su32(&bar)), "r"(other));
    for (int r = 0; r < rounds; ++r) {
      if (rank == 0) asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
      asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(&bar)), "r"((unsigned)(r & 1)) : "memory");
      if (rank != 0) asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
    }
  }
  long long t1 = clock64();
  cl.sync();
  long long t2 = clock64();
  if (active) {   // (ii) DSMEM flag ping-pong
    volatile unsigned* rf = cl.map_shared_rank((unsigned*)&flag, other);
    for (int r = 1; r <= rounds; ++r) {
      if (rank == 0) *rf = r;
      while (flag != (unsigned)r) {}
      if (rank != 0) *rf = r;
    }
  }
  long long t3 = clock64();
  cl.sync();
  long long t4 = clock64();
  for (int r = 0; r < rounds; ++r) cl.sync();   // (iii) cluster barrier (all threads)
  long long t5 = clock64();
  if (rank == 0 && threadIdx.x == 0) {
    out[0] = t1 - t0;
    out[1] = t3 - t2;
    out[2] = t5 - t4;
  }
}
int main() {
  long long* out; cudaMalloc(&out, 64);
  const int rounds = 1000;
  for (int peer : {1, 4, 7}) {
    for (int rep = 0; rep < 2; ++rep) k_pp<<<8, 256>>>(rounds, peer, out);
    cudaDeviceSynchronize();
    long long h[3]; cudaMemcpy(h, out, 24, cudaMemcpyDeviceToHost);
    printf("peer %d: mbarrier remote-arrive round trip %.0f cycles, DSMEM flag round trip %.0f, cluster.sync %.0f\n",
           peer, (double)h[0] / rounds, (double)h[1] / rounds, (double)h[2] / rounds);
  }
  return 0;
}
