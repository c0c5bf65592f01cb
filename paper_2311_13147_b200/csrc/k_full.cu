// NEXT-2: the two-stage Sinkhorn algorithm for C-EROT with approximate cyclic symmetry
// (Algorithm 3). Stage 1 is the cyclic Sinkhorn of the hot path on the fold averages (lines 2-10);
// stage 2 (lines 11-16) is the original Sinkhorn on the explicit d x d problem, here WITHOUT materialising
// the d x d cost: C is block-circulant (Assumption 1 holds for C strictly), so the row I = r*m + i
// of the explicit cost is the n block rows C_k[i][:] permuted by r (entry J = s*m + j is C_{(s-r) mod n}[i][j],
// P:161-168). One CTA per i stages those n*m values in shared memory once and serves all n rows r from them
// (n-fold reuse on chip); the column half-iteration is the same kernel on the transposed blocks
// B_k = C_{(-k) mod n}^T (the transpose of a block-circulant matrix is block-circulant).
//
// Potentials are eps-scaled and fp64 (f_hat = f/eps, g_hat = g/eps, d = n*m each). Per element the argument
// x = in_J - X_IJ/eps is fp64; the exponential is MUFU.EX2 with the exact exponent split (fp32 costs) or the
// fp64 exp (fp64 costs), after the row maximum (two passes over the row, no overflow).
#include "common.cuh"
#include "internal.h"

namespace cot {

// alpha_i = (1/n) sum_k a_{i + m k}, beta likewise (Alg. 3 lines 2-5).
__global__ void k_fold(const double* __restrict__ a, const double* __restrict__ b, int64_t n, int64_t m,
                       double* __restrict__ alpha, double* __restrict__ beta) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double sa = 0.0, sb = 0.0;
  for (int64_t k = 0; k < n; ++k) {
    sa += a[i + m * k];
    sb += b[i + m * k];
  }
  alpha[i] = sa / (double)n;
  beta[i] = sb / (double)n;
}

// g_hat = the n concatenated z_hat (Alg. 3 line 11: q = concatenated q^).
__global__ void k_tile(const double* __restrict__ z, int64_t n, int64_t m, double* __restrict__ g) {
  const int64_t J = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (J < n * m) g[J] = z[J % m];
}

// B_k[j][i] = C_{(n - k) mod n}[i][j]: the blocks of the transposed block-circulant matrix.
template <typename T>
__global__ void k_transpose_blocks(const T* __restrict__ C, int64_t n, int64_t m, T* __restrict__ Bt) {
  __shared__ T tile[32][33];
  const int64_t k = blockIdx.z;
  const int64_t src = (n - k) % n;
  const int64_t i0 = (int64_t)blockIdx.y * 32, j0 = (int64_t)blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + r, j = j0 + threadIdx.x;
    if (i < m && j < m) tile[r][threadIdx.x] = C[(src * m + i) * m + j];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t j = j0 + r, i = i0 + threadIdx.x;
    if (i < m && j < m) Bt[(k * m + j) * m + i] = tile[threadIdx.x][r];
  }
}

template <typename T>
__device__ __forceinline__ double exp_arg(double x);
template <>
__device__ __forceinline__ double exp_arg<double>(double x) { return exp(x); }
template <>
__device__ __forceinline__ double exp_arg<float>(double x) {   // e^x, x <= ~0: exact 2^round, MUFU 2^frac
  const double a = x * COT_LOG2E;
  const double big = a + 6755399441055744.0;   // round to nearest integer (|a| < 2^51)
  const int ai = max(__double2loint(big), -1022);
  return (double)ex2((float)(a - (big - 6755399441055744.0))) * __hiloint2double((ai + 1023) << 20, 0);
}

__device__ __forceinline__ double blk_reduce(double v, bool is_max, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = is_max ? warp_max(v) : warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = sh[0];
  for (int w = 1; w < nw; ++w) t = is_max ? fmax(t, sh[w]) : t + sh[w];
  return t;
}

// One half-iteration of stage 2 over the block-circulant matrix with blocks X [n][m][m]:
//   out_I = log mu_I - LSE_J (in_J - X_IJ / eps),  I = r*m + i,  X_IJ = X_{(s - r) mod n}[i][j], J = s*m + j.
// mode 0: out = the new potential. mode 1 (column half, monitor): also dev_I = |exp(out_old_I + LSE) - mu_I|,
// the column residual of the row-exact plan. mode 2 (report): row sums r_I, transport and
// entropy terms of T_IJ = exp(in_J + out_I - X_IJ/eps) with out read, not written.
// grid = m (one CTA per i), 256 threads; X rows staged in shared memory when they fit (xs != 0). The loops
// run over the column block s (block k = (s - r) mod n) and then j, so no division in the inner loop.
template <typename T>
__global__ void __launch_bounds__(256) k_full_pass(const T* __restrict__ X, int n, int m,
                                                   const double* __restrict__ eps, const double* __restrict__ mu,
                                                   const double* __restrict__ in, double* __restrict__ out,
                                                   double* __restrict__ dev, double* __restrict__ rep, int mode,
                                                   int xs) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* row = reinterpret_cast<T*>(smem_raw);   // [n][m] when xs
  __shared__ double sh[32];
  const int i = blockIdx.x;
  const double inv_eps = 1.0 / eps[0];
  if (xs)
    for (int k = 0; k < n; ++k)
      for (int j = threadIdx.x; j < m; j += blockDim.x) row[(size_t)k * m + j] = X[((size_t)k * m + i) * m + j];
  __syncthreads();
  auto xrow = [&](int k) -> const T* { return xs ? row + (size_t)k * m : X + ((size_t)k * m + i) * m; };
  for (int r = 0; r < n; ++r) {
    const int I = r * m + i;
    if (mode < 2) {
      double mx = -INFINITY;
      for (int s = 0; s < n; ++s) {
        const T* xr = xrow(s >= r ? s - r : s - r + n);
        const double* ir = in + (size_t)s * m;
        for (int j = threadIdx.x; j < m; j += blockDim.x) mx = fmax(mx, ir[j] - (double)xr[j] * inv_eps);
      }
      mx = blk_reduce(mx, true, sh);
      double sum = 0.0;
      for (int s = 0; s < n; ++s) {
        const T* xr = xrow(s >= r ? s - r : s - r + n);
        const double* ir = in + (size_t)s * m;
        for (int j = threadIdx.x; j < m; j += blockDim.x) sum += exp_arg<T>(ir[j] - (double)xr[j] * inv_eps - mx);
      }
      sum = blk_reduce(sum, false, sh);
      if (threadIdx.x == 0) {
        const double lse = mx + log(sum);
        if (mode == 1) dev[I] = fabs(exp(out[I] + lse) - mu[I]);
        out[I] = log(mu[I]) - lse;
      }
    } else {
      const double o = out[I];
      double rs = 0.0, tr = 0.0, en = 0.0;
      for (int s = 0; s < n; ++s) {
        const T* xr = xrow(s >= r ? s - r : s - r + n);
        const double* ir = in + (size_t)s * m;
        for (int j = threadIdx.x; j < m; j += blockDim.x) {
          const double c = (double)xr[j];
          const double lt = ir[j] + o - c * inv_eps;   // log T_IJ
          const double t = exp(lt);
          rs += t;
          tr += c * t;
          en += t * (lt - 1.0);
        }
      }
      rs = blk_reduce(rs, false, sh);
      tr = blk_reduce(tr, false, sh);
      en = blk_reduce(en, false, sh);
      if (threadIdx.x == 0) {
        rep[3 * I + 0] = rs;
        rep[3 * I + 1] = tr;
        rep[3 * I + 2] = en;
      }
    }
  }
}

// Monitor of stage 2: the full problem's column residual sum_J dev_J (fixed order).
__global__ void k_full_monitor(const double* __restrict__ dev, int64_t d, double* __restrict__ out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int64_t J = threadIdx.x; J < d; J += blockDim.x) s += dev[J];
  s = blk_reduce(s, false, sh);
  if (threadIdx.x == 0) out[0] = s;
}

// Report of the stage-2 plan (cot_report order, FULL problem: no factor n): from the row pass (rep_rows:
// r_I, transport_I, entropy_I) and the column pass on the transposed blocks (rep_cols: c_J, ...).
__global__ void k_full_finalize(const double* __restrict__ rep_rows, const double* __restrict__ rep_cols,
                                const double* __restrict__ a, const double* __restrict__ b,
                                const double* __restrict__ f, const double* __restrict__ g, int64_t d,
                                const double* __restrict__ eps, double residual, double* __restrict__ report) {
  __shared__ double sh[32];
  double tr = 0.0, en = 0.0, mass = 0.0, rl1 = 0.0, cl1 = 0.0, cl2 = 0.0, dual = 0.0;
  for (int64_t I = threadIdx.x; I < d; I += blockDim.x) {
    tr += rep_rows[3 * I + 1];
    en += rep_rows[3 * I + 2];
    mass += rep_rows[3 * I + 0];
    rl1 += fabs(rep_rows[3 * I + 0] - a[I]);
    const double dc = rep_cols[3 * I + 0] - b[I];
    cl1 += fabs(dc);
    cl2 += dc * dc;
    dual += f[I] * a[I] + g[I] * b[I];
  }
  tr = blk_reduce(tr, false, sh);
  en = blk_reduce(en, false, sh);
  mass = blk_reduce(mass, false, sh);
  rl1 = blk_reduce(rl1, false, sh);
  cl1 = blk_reduce(cl1, false, sh);
  cl2 = blk_reduce(cl2, false, sh);
  dual = blk_reduce(dual, false, sh);
  if (threadIdx.x == 0) {
    const double e = eps[0];
    report[0] = tr;                     // transport cost <C, T>
    report[1] = tr + e * en;            // regularised primal
    report[2] = e * (dual - mass);      // dual <f,a> + <g,b> - eps sum T (P:358-360 with n = 1)
    report[3] = rl1;
    report[4] = cl1;
    report[5] = sqrt(cl2);
    report[6] = mass;
    report[7] = residual;
  }
}

cudaError_t launch_fold(const double* a, const double* b, int64_t n, int64_t m, double* alpha, double* beta,
                        cudaStream_t s) {
  k_fold<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(a, b, n, m, alpha, beta);
  return cudaGetLastError();
}

cudaError_t launch_tile(const double* z, int64_t n, int64_t m, double* g, cudaStream_t s) {
  k_tile<<<(unsigned)((n * m + 255) / 256), 256, 0, s>>>(z, n, m, g);
  return cudaGetLastError();
}

cudaError_t launch_transpose_blocks(const void* C, int64_t n, int64_t m, int dtype, void* Bt, cudaStream_t s) {
  dim3 grid((unsigned)((m + 31) / 32), (unsigned)((m + 31) / 32), (unsigned)n), block(32, 8);
  if (dtype == COT_F32)
    k_transpose_blocks<float><<<grid, block, 0, s>>>(static_cast<const float*>(C), n, m, static_cast<float*>(Bt));
  else
    k_transpose_blocks<double><<<grid, block, 0, s>>>(static_cast<const double*>(C), n, m, static_cast<double*>(Bt));
  return cudaGetLastError();
}

cudaError_t launch_full_pass(const void* X, int64_t n, int64_t m, int dtype, const double* eps, const double* mu,
                             const double* in, double* out, double* dev, double* rep, int mode, cudaStream_t s) {
  const size_t esz = dtype == COT_F32 ? 4 : 8;
  const size_t bytes = (size_t)n * m * esz;
  const int xs = bytes <= 96 * 1024 ? 1 : 0;
  const size_t smem = xs ? bytes : 0;
  cudaError_t e;
  if (dtype == COT_F32) {
    e = cudaFuncSetAttribute(k_full_pass<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_full_pass<float><<<(unsigned)m, 256, smem, s>>>(static_cast<const float*>(X), (int)n, (int)m, eps, mu, in, out,
                                                      dev, rep, mode, xs);
  } else {
    e = cudaFuncSetAttribute(k_full_pass<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_full_pass<double><<<(unsigned)m, 256, smem, s>>>(static_cast<const double*>(X), (int)n, (int)m, eps, mu, in,
                                                       out, dev, rep, mode, xs);
  }
  return cudaGetLastError();
}

cudaError_t launch_full_monitor(const double* dev, int64_t d, double* out, cudaStream_t s) {
  k_full_monitor<<<1, 1024, 0, s>>>(dev, d, out);
  return cudaGetLastError();
}

cudaError_t launch_full_finalize(const double* rep_rows, const double* rep_cols, const double* a, const double* b,
                                 const double* f, const double* g, int64_t d, const double* eps, double residual,
                                 double* report, cudaStream_t s) {
  k_full_finalize<<<1, 1024, 0, s>>>(rep_rows, rep_cols, a, b, f, g, d, eps, residual, report);
  return cudaGetLastError();
}

}  // namespace cot
