// NEXT-3: C-SROT with the squared regulariser phi(x) = x^2/(2 gamma) (x >= 0) through the 2m-variable Fenchel
// dual (Theorem 2) and alternating maximisation: with z fixed, every w_i solves
//     alpha_i = sum_{j,k} (phi*)'(w_i + z_j - C_ijk) = gamma sum_{j,k} max(w_i + z_j - C_ijk, 0)
// (eq. derivative_of_objective_function), and symmetrically for z_j with w fixed. The right side
// is convex, increasing and piecewise linear in w_i with breakpoints b = C_ijk - z_j, so Newton started to
// the right of the root (w = min b + alpha_i/gamma) decreases monotonically to it in finitely many steps;
// every Newton step is one streamed pass over the row's n*m costs. Sums are not factorisable over k (unlike
// the entropic case), so the n*m^2 stream per pass is inherent.
#include "common.cuh"
#include "internal.h"

#include <algorithm>

namespace cot {

__device__ __forceinline__ void blk_sum2(double& a, double& b, double* sh, int& buf) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  double* r = sh + buf * 64;
  if (lane == 0) {
    r[wid] = a;
    r[32 + wid] = b;
  }
  __syncthreads();
  double A = 0.0, B2 = 0.0;
  for (int w = 0; w < nw; ++w) {
    A += r[w];
    B2 += r[32 + w];
  }
  a = A;
  b = B2;
  buf ^= 1;
}
__device__ __forceinline__ double blk_min(double v, double* sh, int& buf) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  double* r = sh + buf * 64;
  if (lane == 0) r[wid] = v;
  __syncthreads();
  double t = r[0];
  for (int w = 1; w < nw; ++w) t = fmin(t, r[w]);
  buf ^= 1;
  return t;
}

// w-step: one CTA per (problem, row).
template <typename T>
__global__ void __launch_bounds__(256) k_srot_rows(const T* __restrict__ C, const double* __restrict__ alpha,
                                                   const double* __restrict__ z, double* __restrict__ w,
                                                   const double* __restrict__ gam, int64_t B, int64_t n, int64_t m,
                                                   const SolverState* __restrict__ state) {
  __shared__ double sh[128];
  extern __shared__ double zs[];   // [m] z of the current problem
  int buf = 0;
  int64_t zb = -1;
  for (int64_t u = blockIdx.x; u < B * m; u += gridDim.x) {
    const int64_t b = u / m, i = u - b * m;
    if (!state[b].active) continue;
    if (b != zb) {   // block-uniform
      __syncthreads();
      for (int64_t j = threadIdx.x; j < m; j += blockDim.x) zs[j] = z[b * m + j];
      __syncthreads();
      zb = b;
    }
    const double g = gam[b];
    const double A = alpha[b * m + i] / g;
    const T* Cb = C + b * n * m * m + i * m;                       // C[b][k][i][j] = Cb[k*m*m + j]
    double lmin = INFINITY;
    for (int64_t k = 0; k < n; ++k)
      for (int64_t j = threadIdx.x; j < m; j += blockDim.x) lmin = fmin(lmin, (double)Cb[k * m * m + j] - zs[j]);
    const double bmin = blk_min(lmin, sh, buf);
    double x = bmin + A;                                           // right of the root
    for (int it = 0; it < 200; ++it) {
      double S = 0.0, N = 0.0;
      for (int64_t k = 0; k < n; ++k)
        for (int64_t j = threadIdx.x; j < m; j += blockDim.x) {
          const double d = x - ((double)Cb[k * m * m + j] - zs[j]);
          if (d > 0.0) {
            S += d;
            N += 1.0;
          }
        }
      blk_sum2(S, N, sh, buf);
      const double F = S - A;                                      // >= 0 (convex, from the right)
      if (F <= 1e-14 * A || N == 0.0) break;
      x -= F / N;
    }
    if (threadIdx.x == 0) w[b * m + i] = x;
  }
}

// z-step: a block owns TW = 4 consecutive columns; thread t handles column t % TW and the (k, i) pairs
// (t / TW) + q * (256 / TW) -- 64 partial sums per column, combined in a fixed order (deterministic). All
// columns of the tile iterate their Newton steps together. The first evaluation at the old z gives the plan's
// column sums c_j (monitor). grid = (ceil(m / TW), B).
constexpr int kSrotTW = 4;
template <typename T>
__global__ void __launch_bounds__(256) k_srot_cols(const T* __restrict__ C, const double* __restrict__ beta,
                                                   const double* __restrict__ w, double* __restrict__ z,
                                                   const double* __restrict__ gam, int64_t n, int64_t m,
                                                   double* __restrict__ resid_part, SolverState* __restrict__ state,
                                                   unsigned* __restrict__ counters, double tol, int64_t check_every) {
  constexpr int TW = kSrotTW, NG = 256 / TW;
  const int64_t b = blockIdx.y;
  const int ntiles = gridDim.x;
  if (!state[b].active) return;
  const int c = threadIdx.x % TW, grp = threadIdx.x / TW;
  const int64_t j = (int64_t)blockIdx.x * TW + c;
  const bool ok = j < m;
  __shared__ double sS[NG][TW], sN[NG][TW];
  __shared__ int any_active;
  __shared__ bool is_last;
  const double g = gam[b];
  const double Bt = ok ? beta[b * m + j] / g : 0.0;
  const T* Cb = C + b * n * m * m;
  auto reduce = [&](double& S, double& N, bool is_min) {
    sS[grp][c] = S;
    sN[grp][c] = N;
    __syncthreads();
    double a0 = sS[0][c], a1 = sN[0][c];
    for (int q = 1; q < NG; ++q) {
      a0 = is_min ? fmin(a0, sS[q][c]) : a0 + sS[q][c];
      a1 += sN[q][c];
    }
    __syncthreads();
    S = a0;
    N = a1;
  };
  extern __shared__ double ws_[];   // [m] w of this problem
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) ws_[i] = w[b * m + i];
  __syncthreads();
  auto pass = [&](double x, double& S, double& N) {
    S = 0.0;
    N = 0.0;
    if (ok)
      for (int64_t k = 0; k < n; ++k) {
        const T* Ck = Cb + k * m * m + j;
        int64_t i = grp;
        for (; i + 3 * NG < m; i += 4 * NG) {   // 4 loads in flight
          T cv[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) cv[q] = Ck[(i + q * NG) * m];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double d = x - ((double)cv[q] - ws_[i + q * NG]);
            if (d > 0.0) {
              S += d;
              N += 1.0;
            }
          }
        }
        for (; i < m; i += NG) {
          const double d = x - ((double)Ck[i * m] - ws_[i]);
          if (d > 0.0) {
            S += d;
            N += 1.0;
          }
        }
      }
    reduce(S, N, false);
  };
  // monitor: column sums of the plan after the w-step, at the old z
  const double zold = ok ? z[b * m + j] : 0.0;
  double S0, N0;
  pass(zold, S0, N0);
  const double cj = g * S0;
  const double dev = ok && grp == 0 ? fabs(cj - beta[b * m + j]) : 0.0;
  // minimum breakpoint of this column
  double lmin = INFINITY, dummy = 0.0;
  if (ok)
    for (int64_t k = 0; k < n; ++k)
      for (int64_t i = grp; i < m; i += NG) lmin = fmin(lmin, (double)Cb[(k * m + i) * m + j] - ws_[i]);
  reduce(lmin, dummy, true);
  double x = lmin + Bt;
  bool act = ok;
  for (int it = 0; it < 200; ++it) {
    double S, N;
    pass(x, S, N);
    const double F = S - Bt;
    if (act && (F <= 1e-14 * Bt || N == 0.0)) act = false;
    if (act) x -= F / N;
    if (threadIdx.x == 0) any_active = 0;
    __syncthreads();
    if (act) any_active = 1;
    __syncthreads();
    if (!any_active) break;
  }
  if (ok && grp == 0) z[b * m + j] = x;
  // monitor reduction (per block in column order, then last block per problem in block order) + freeze rule
  __shared__ double sdev[TW];
  if (grp == 0) sdev[c] = dev;
  __syncthreads();
  if (threadIdx.x == 0) {
    double d = 0.0;
    for (int q = 0; q < TW; ++q) d += sdev[q];
    resid_part[b * ntiles + blockIdx.x] = d;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(&counters[b], 1u) == (unsigned)(ntiles - 1);
  __syncthreads();
  if (is_last && threadIdx.x == 0) {
    __threadfence();
    double r = 0.0;
    for (int t = 0; t < ntiles; ++t) r += __ldcg(resid_part + b * ntiles + t);
    r *= (double)n;
    SolverState& st = state[b];
    st.residual = r;
    st.iters += 1;
    if (tol > 0.0 && st.iters % check_every == 0 && r <= tol) {
      st.active = 0;
      st.converged = 1;
    }
    counters[b] = 0u;
  }
}

// Column sums c_j of the plan gamma max(w_i + z_j - C_ijk, 0) for the report (same tile layout as the z-step).
template <typename T>
__global__ void __launch_bounds__(256) k_srot_colsum(const T* __restrict__ C, const double* __restrict__ w,
                                                     const double* __restrict__ z, const double* __restrict__ gam,
                                                     int64_t n, int64_t m, double* __restrict__ colsum) {
  constexpr int TW = kSrotTW, NG = 256 / TW;
  const int64_t b = blockIdx.y;
  const int c = threadIdx.x % TW, grp = threadIdx.x / TW;
  const int64_t j = (int64_t)blockIdx.x * TW + c;
  __shared__ double sS[NG][TW];
  double S = 0.0;
  if (j < m) {
    const double zj = z[b * m + j];
    const T* Cb = C + b * n * m * m;
    for (int64_t l = grp; l < n * m; l += NG) {
      const int64_t k = l / m, i = l - k * m;
      const double y = w[b * m + i] + zj - (double)Cb[(k * m + i) * m + j];
      S += y > 0.0 ? y : 0.0;
    }
  }
  sS[grp][c] = S;
  __syncthreads();
  if (grp == 0 && j < m) {
    double t = 0.0;
    for (int q = 0; q < NG; ++q) t += sS[q][c];
    colsum[b * m + j] = gam[b] * t;
  }
}

// Plan T_ijk = gamma max(w_i + z_j - C_ijk, 0) (eq. optimality_condition) and the report:
// per (problem, row) CTA: transport, sum phi(T), sum phi*(w+z-C), row residual; column sums into buf.
template <typename T>
__global__ void __launch_bounds__(256) k_srot_plan(const T* __restrict__ C, const double* __restrict__ w,
                                                   const double* __restrict__ z, const double* __restrict__ alpha,
                                                   const double* __restrict__ gam, int64_t B, int64_t n, int64_t m,
                                                   T* __restrict__ Tout, double* __restrict__ rowscal,
                                                   double* __restrict__ colsum) {
  __shared__ double sh[128];
  int buf = 0;
  for (int64_t u = blockIdx.x; u < B * m; u += gridDim.x) {
    const int64_t b = u / m, i = u - b * m;
    const double g = gam[b];
    const double wi = w[b * m + i];
    double tr = 0.0, ph = 0.0, cj = 0.0, row = 0.0;
    for (int64_t l = threadIdx.x; l < n * m; l += blockDim.x) {
      const int64_t k = l / m, j = l - k * m;
      const int64_t idx = ((b * n + k) * m + i) * m + j;
      const double c = (double)C[idx];
      const double y = wi + z[b * m + j] - c;
      const double t = y > 0.0 ? g * y : 0.0;
      if (Tout) Tout[idx] = (T)t;
      tr += c * t;
      ph += t * t / (2.0 * g);
      cj += y > 0.0 ? 0.5 * g * y * y : 0.0;
      row += t;
    }
    blk_sum2(tr, ph, sh, buf);
    blk_sum2(cj, row, sh, buf);
    if (threadIdx.x == 0) {
      double* o = rowscal + u * 4;
      o[0] = tr;
      o[1] = ph;
      o[2] = cj;
      o[3] = row;
    }
  }
  (void)colsum;
}

// One block per problem: column sums (fixed order over rows) and the report.
template <typename T>
__global__ void __launch_bounds__(256) k_srot_finalize(const T* __restrict__ C, const double* __restrict__ w,
                                                       const double* __restrict__ z,
                                                       const double* __restrict__ alpha,
                                                       const double* __restrict__ beta,
                                                       const double* __restrict__ gam, const double* __restrict__ rowscal,
                                                       const double* __restrict__ colsum, int64_t n, int64_t m,
                                                       const SolverState* __restrict__ state,
                                                       double* __restrict__ report) {
  __shared__ double sh[128];
  int buf = 0;
  const int64_t b = blockIdx.x;
  const double g = gam[b];
  (void)C;
  (void)g;
  double cl1 = 0.0, cl2 = 0.0;
  for (int64_t j = threadIdx.x; j < m; j += blockDim.x) {
    const double dv = colsum[b * m + j] - beta[b * m + j];
    cl1 += fabs(dv);
    cl2 += dv * dv;
  }
  blk_sum2(cl1, cl2, sh, buf);
  double dot = 0.0, rl1 = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    dot += w[b * m + i] * alpha[b * m + i] + z[b * m + i] * beta[b * m + i];
    rl1 += fabs(rowscal[(b * m + i) * 4 + 3] - alpha[b * m + i]);
  }
  blk_sum2(dot, rl1, sh, buf);
  if (threadIdx.x == 0) {
    double tr = 0.0, ph = 0.0, cj = 0.0, mass = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      const double* o = rowscal + (b * m + i) * 4;
      tr += o[0];
      ph += o[1];
      cj += o[2];
      mass += o[3];
    }
    const double nn = (double)n;
    double* rep = report + b * kReportDoubles;
    rep[0] = nn * tr;                 // transport cost of the full plan
    rep[1] = nn * (tr + ph);          // regularised primal
    rep[2] = nn * (dot - cj);         // dual
    rep[3] = nn * rl1;
    rep[4] = nn * cl1;
    rep[5] = sqrt(nn * cl2);
    rep[6] = nn * mass;
    rep[7] = state ? state[b].residual : 0.0;
  }
}

cudaError_t launch_srot_sweep(const IterArgs& a, const double* gam, const Workspace& ws, cudaStream_t s) {
  const int sms = device_sm_count();
  const int64_t rows = a.B * a.m;
  const int grid = (int)std::min<int64_t>(rows, (int64_t)sms * 8);
  dim3 cgrid((unsigned)((a.m + kSrotTW - 1) / kSrotTW), (unsigned)a.B);
  const size_t zbytes = (size_t)a.m * 8;   // z (w-step) or w (z-step) of one problem in shared memory
  if (zbytes > 48 * 1024) return cudaErrorInvalidValue;
  if (a.dtype == COT_F32) {
    k_srot_rows<float><<<grid, 256, zbytes, s>>>((const float*)a.C, a.alpha, a.z_hat, a.w_hat, gam, a.B, a.n, a.m, ws.state);
    k_srot_cols<float><<<cgrid, 256, zbytes, s>>>((const float*)a.C, a.beta, a.w_hat, a.z_hat, gam, a.n, a.m, ws.resid_part,
                                             ws.state, ws.counters, a.tol, a.check_every);
  } else {
    k_srot_rows<double><<<grid, 256, zbytes, s>>>((const double*)a.C, a.alpha, a.z_hat, a.w_hat, gam, a.B, a.n, a.m,
                                             ws.state);
    k_srot_cols<double><<<cgrid, 256, zbytes, s>>>((const double*)a.C, a.beta, a.w_hat, a.z_hat, gam, a.n, a.m,
                                              ws.resid_part, ws.state, ws.counters, a.tol, a.check_every);
  }
  return cudaGetLastError();
}

cudaError_t launch_srot_plan(const IterArgs& a, const double* gam, const Workspace& ws, void* T_blocks,
                             double* report, cudaStream_t s) {
  const int sms = device_sm_count();
  const int64_t rows = a.B * a.m;
  const int grid = (int)std::min<int64_t>(rows, (int64_t)sms * 8);
  double* rowscal = ws.rowscal;       // [B*m][4]
  double* colsum = ws.c_local;        // [B][m]
  dim3 cgrid((unsigned)((a.m + kSrotTW - 1) / kSrotTW), (unsigned)a.B);
  if (a.dtype == COT_F32) {
    k_srot_plan<float><<<grid, 256, 0, s>>>((const float*)a.C, a.w_hat, a.z_hat, a.alpha, gam, a.B, a.n, a.m,
                                            (float*)T_blocks, rowscal, nullptr);
    k_srot_colsum<float><<<cgrid, 256, 0, s>>>((const float*)a.C, a.w_hat, a.z_hat, gam, a.n, a.m, colsum);
    k_srot_finalize<float><<<(unsigned)a.B, 256, 0, s>>>((const float*)a.C, a.w_hat, a.z_hat, a.alpha, a.beta, gam,
                                                         rowscal, colsum, a.n, a.m, ws.state, report);
  } else {
    k_srot_plan<double><<<grid, 256, 0, s>>>((const double*)a.C, a.w_hat, a.z_hat, a.alpha, gam, a.B, a.n, a.m,
                                             (double*)T_blocks, rowscal, nullptr);
    k_srot_colsum<double><<<cgrid, 256, 0, s>>>((const double*)a.C, a.w_hat, a.z_hat, gam, a.n, a.m, colsum);
    k_srot_finalize<double><<<(unsigned)a.B, 256, 0, s>>>((const double*)a.C, a.w_hat, a.z_hat, a.alpha, a.beta, gam,
                                                          rowscal, colsum, a.n, a.m, ws.state, report);
  }
  return cudaGetLastError();
}

}  // namespace cot
