// Microbenchmark: dependent-chain latencies (cycles) of the instruction classes in the epilogue critical path.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k_lat(double* out, long long* cyc, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9;
  float f = (float)a;
  __shared__ double sh[64];
  sh[threadIdx.x & 63] = a;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (OP == 0) a = a + 1.0000001;                                   // DADD
    if (OP == 1) a = fma(a, 0.9999999, 1e-9);                         // DFMA
    if (OP == 2) { f = (float)a; a = (double)f; }                     // F2F pair
    if (OP == 3) { asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(f) : "f"(f)); f = f * 0.5f; }  // MUFU + FMUL
    if (OP == 4) a = __shfl_xor_sync(0xffffffffu, a, 1);              // SHFL (double = 2 SHFL)
    if (OP == 5) { asm volatile("bar.sync 1, %0;" ::"r"((int)blockDim.x)); a += 1.0; }   // bar.sync + DADD
    if (OP == 6) a = sh[((int)a) & 63] + 1.0;                          // LDS.64 + DADD
    if (OP == 7) a = log(a) + 2.0;                                     // fp64 log
    if (OP == 8) a = exp(-a) + 1.0;                                    // fp64 exp
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + f;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 1024);
  const char* names[] = {"DADD", "DFMA", "F2F f64>f32>f64", "MUFU.EX2+FMUL", "SHFL f64", "bar.sync(256)+DADD", "LDS.64+DADD",
                         "log() f64 + DADD", "exp() f64 + DADD"};
  void (*fns[])(double*, long long*, int, double) = {k_lat<0>, k_lat<1>, k_lat<2>, k_lat<3>, k_lat<4>, k_lat<5>, k_lat<6>,
                                                     k_lat<7>, k_lat<8>};
  const int iters = 4096;
  for (int o = 0; o < 9; ++o) {
    for (int threads : {32, 256}) {
      long long h = 0;
      for (int rep = 0; rep < 2; ++rep) {
        fns[o]<<<1, threads>>>(out, cyc, iters, 0.5);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      }
      printf("%-22s threads=%3d: %.1f cycles per dependent op\n", names[o], threads, (double)h / iters);
    }
  }
  return 0;
}
