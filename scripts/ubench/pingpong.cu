// Microbenchmark: one-way latency of an LL line (16-byte volatile store -> volatile polling load) between two
// CTAs of one launch on different SMs, via L2. Block 0 pings, block `peer` pongs; all other blocks exit.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void st_line(uint4* p, uint4 v) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ uint4 ld_line(const uint4* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__global__ void k_pp(uint4* lines, int peer, int rounds, long long* out, unsigned* smid) {
  unsigned id;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
  if (threadIdx.x == 0) smid[blockIdx.x] = id;
  if (threadIdx.x != 0 || (blockIdx.x != 0 && blockIdx.x != (unsigned)peer)) return;
  const bool ping = blockIdx.x == 0;
  uint4* mine = lines + (ping ? 0 : 1);
  uint4* theirs = lines + (ping ? 1 : 0);
  const long long t0 = clock64();
  for (unsigned g = 1; g <= (unsigned)rounds; ++g) {
    if (ping) {
      st_line(mine, make_uint4(g, g, g, g));
      while (ld_line(theirs).y != g) {}
    } else {
      while (ld_line(theirs).y != g) {}
      st_line(mine, make_uint4(g, g, g, g));
    }
  }
  if (ping) out[0] = clock64() - t0;
}
int main() {
  uint4* lines; long long* out; unsigned* smid;
  cudaMalloc(&lines, 4096); cudaMalloc(&out, 8); cudaMalloc(&smid, 4096);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int rounds = 2000;
  for (int peer : {1, 2, 8, 37, 74, 100, 147}) {
    cudaMemset(lines, 0, 4096);
    void* args[] = {&lines, &peer, (void*)&rounds, &out, &smid};
    int r = rounds;
    args[2] = &r;
    cudaLaunchCooperativeKernel((void*)k_pp, dim3(sms), dim3(32), args, 0, 0);
    cudaDeviceSynchronize();
    long long h; unsigned s[148];
    cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(s, smid, sms * 4, cudaMemcpyDeviceToHost);
    printf("peer block %3d (SM %3u vs SM %3u): %.0f cycles per round trip (%.0f one way)\n", peer, s[0], s[peer],
           (double)h / rounds, (double)h / rounds / 2);
  }
  return 0;
}
