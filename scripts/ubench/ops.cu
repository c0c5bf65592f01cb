// Microbenchmark: per-SM throughput of the instruction classes of the C-EROT epilogue on this GPU
// (DADD, DFMA, F2F f64->f32, F2F f32->f64, MUFU.EX2, SHFL of a double), 16 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k_op(double* out, int iters, double seed) {
  double a[16];
  float f[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    a[i] = 1e-3 * (threadIdx.x + i) + seed;
    f[i] = (float)a[i];
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (OP == 0) a[i] = a[i] + 1.0000001;                       // DADD
      if (OP == 1) a[i] = fma(a[i], 0.9999999, 1e-7);             // DFMA
      if (OP == 2) { f[i] = (float)a[i]; a[i] = (double)f[i] * 0.5; }   // F2F pair (+DMUL)
      if (OP == 3) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(f[i])); f[i] = y - 1.0f; }
      if (OP == 4) a[i] += __shfl_xor_sync(0xffffffffu, a[i], 1 + (i & 7));
      if (OP == 5) a[i] = a[i] * 0.9999999;                       // DMUL
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i] + f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out; cudaMalloc(&out, sms * 2 * 1024 * 8);
  const int iters = 2048;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"DADD", "DFMA", "F2F pair+DMUL", "MUFU.EX2", "SHFL.f64+DADD", "DMUL"};
  void (*fns[])(double*, int, double) = {k_op<0>, k_op<1>, k_op<2>, k_op<3>, k_op<4>, k_op<5>};
  for (int o = 0; o < 6; ++o)
    for (int threads : {128, 512}) {
      float ms = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        fns[o]<<<sms, threads>>>(out, iters, 0.5);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      double ops = (double)sms * threads * iters * 16;
      printf("%-16s threads=%4d: %.2f per SM per clk (@%d MHz max)\n", names[o], threads, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  return 0;
}
