// Microbenchmark: the k-sum inner loop of the cluster-resident kernel in isolation (float4 from shared
// memory, FFMA + MUFU.EX2 + FADD per element), one CTA per SM, W warps, R rows per warp: ex2 per SM per clk.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
template <int MODE>
__global__ void k_ksum(float* out, int iters, int n, int rows_per_warp) {
  extern __shared__ float4 cs[];   // [rows][n][32] float4
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int total = nw * rows_per_warp * n * 32;
  for (int i = threadIdx.x; i < total; i += blockDim.x)
    cs[i] = make_float4(0.01f * (i & 7), 0.02f * (i & 3), 0.03f, 0.04f);
  __syncthreads();
  const float c2 = 1.7f, g = 0.3f;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    for (int rr = 0; rr < rows_per_warp; ++rr) {
      const float4* crow = cs + (size_t)(warp + rr * nw) * n * 32;
      float s0 = 0, s1 = 0, s2 = 0, s3 = 0;
      for (int k = 0; k < n; k += 4) {
        if (MODE == 0) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const float4 c = crow[(k + kk) * 32 + lane];
            s0 += ex2(fmaf(-c.x, c2, g));
            s1 += ex2(fmaf(-c.y, c2, g));
            s2 += ex2(fmaf(-c.z, c2, g));
            s3 += ex2(fmaf(-c.w, c2, g));
          }
        } else {
          float e[4][4];
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const float4 c = crow[(k + kk) * 32 + lane];
            e[kk][0] = ex2(fmaf(-c.x, c2, g));
            e[kk][1] = ex2(fmaf(-c.y, c2, g));
            e[kk][2] = ex2(fmaf(-c.z, c2, g));
            e[kk][3] = ex2(fmaf(-c.w, c2, g));
          }
          s0 += (e[0][0] + e[1][0]) + (e[2][0] + e[3][0]);
          s1 += (e[0][1] + e[1][1]) + (e[2][1] + e[3][1]);
          s2 += (e[0][2] + e[1][2]) + (e[2][2] + e[3][2]);
          s3 += (e[0][3] + e[1][3]) + (e[2][3] + e[3][3]);
        }
      }
      acc += s0 + s1 + s2 + s3;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, sms * 1024 * 4);
  const int n = 16, iters = 400;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int cfgs[][2] = {{16, 1}, {11, 2}, {8, 2}, {12, 2}, {16, 2}, {4, 4}, {8, 4}};
  for (int mode = 0; mode < 2; ++mode)
    for (auto& c : cfgs) {
      const int W = c[0], R = c[1];
      const size_t smem = (size_t)W * R * n * 32 * 16;
      if (smem > 227 * 1024) continue;
      void* fn = mode ? (void*)k_ksum<1> : (void*)k_ksum<0>;
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        if (mode) k_ksum<1><<<sms, W * 32, smem>>>(out, iters, n, R);
        else k_ksum<0><<<sms, W * 32, smem>>>(out, iters, n, R);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      const double ex = (double)sms * W * R * n * 128 * iters;
      printf("mode %d warps %2d rows/warp %d: %.2f ex2 per SM per clk (@ %d MHz)  %s\n", mode, W, R,
             ex / (best * 1e-3) / sms / (clk * 1e3), clk / 1000, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
