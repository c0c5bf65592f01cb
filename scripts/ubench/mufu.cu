// Microbenchmark: MUFU.EX2 (ex2.approx.ftz.f32) and FFMA throughput per SM on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_ex2(float* out, int iters, float seed) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = -0.001f * (threadIdx.x + i) + seed;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i]));
      a[i] = y - 1.0f;
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma(float* out, int iters, float seed) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = 0.001f * (threadIdx.x + i) + seed;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], 0.999f, 0.0001f);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, sms * 4 * 1024 * 4);
  const int iters = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k_ex2<<<sms * 2, threads>>>(out, iters, 0.5f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)sms * 2 * threads * iters * 16;
      if (rep) printf("ex2  threads/CTA=%4d (2 CTA/SM): %.3e ex2/s = %.2f per SM per clk @ %d MHz (max)\n", threads, ops / (ms * 1e-3), ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
      cudaEventRecord(e0);
      k_ffma<<<sms * 2, threads>>>(out, iters, 0.5f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("ffma threads/CTA=%4d (2 CTA/SM): %.3e ffma/s = %.2f per SM per clk\n", threads, ops / (ms * 1e-3), ops / (ms * 1e-3) / sms / (clk * 1e3));
    }
  }
  return 0;
}
