// K-ITER / K-RED: one cyclic Sinkhorn iteration (Alg. 2 lines 4-5) in the log domain of
// eq. optimal_f_sinkhorn_logdomain, split in two kernels:
//
//  k_rows (row pass, p-update fused with the start of the q-update). For each row i of a unit:
//     s_ij = sum_k exp((G_ij - C_ijk)/eps)     streamed over k: one FFMA + one MUFU.EX2 + one FADD per
//                                              element; G is the exact max of -C/eps => no rescaling
//     x_ij = z_hat_j - G_ij/eps (fp64), M_i = max_j x_ij,  t_ij = s_ij exp(x_ij - M_i),  r_i = sum_j t_ij
//     w_hat_i = log alpha_i - M_i - log r_i                 (the p-update, P:403-411 / P:415)
//     P_uj += (alpha_i / r_i) t_ij                          (plan column mass after the p-update)
//   and writes the unit's fp64 column partial P_u (one row of `partials`).
//  k_cols (column pass): c_j = sum_u P_uj in a fixed order (deterministic), z_hat_j += log beta_j - log c_j
//   (the q-update P:417 in log form), and the monitor n * sum_j |c_j - beta_j| through a
//   last-block-done reduction, plus the convergence/freeze rule.
//
// Work per iteration: n*m^2 Gibbs-kernel evaluations (exp) streamed from HBM, m^2 fp64 epilogue terms.
#include "common.cuh"
#include "internal.h"

namespace cot {

template <typename T, int V>
struct VecL;
template <>
struct VecL<float, 4> {
  using type = float4;
  __device__ static void unpack(const type& v, float* o) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
};
template <>
struct VecL<float, 1> {
  using type = float;
  __device__ static void unpack(const type& v, float* o) { o[0] = v; }
};
template <>
struct VecL<double, 2> {
  using type = double2;
  __device__ static void unpack(const type& v, double* o) { o[0] = v.x; o[1] = v.y; }
};
template <>
struct VecL<double, 1> {
  using type = double;
  __device__ static void unpack(const type& v, double* o) { o[0] = v; }
};

struct RowParams {
  const void* C;         // [B][n][R][m]
  const void* G;         // [B][R][m]
  const double* alpha;   // [B][m] (global rows)
  const double* z_hat;   // [B][m]
  double* w_hat;         // [B][m] (global rows)
  const double* eps;     // [B]
  int64_t n, m, R, row_begin, rpu, upp, U;
  double* partials;      // [U][m]
  const SolverState* state;
  int pre;               // precomputed mode: C is S_ij = sum_k exp((G_ij - C_ijk)/eps) (n = 1), s = S
};

__device__ __forceinline__ double blk_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < nw; ++w) t += sh[w];
  __syncthreads();
  return t;
}
__device__ __forceinline__ double blk_max(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_max(v);
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = sh[0];
  for (int w = 1; w < nw; ++w) t = fmax(t, sh[w]);
  __syncthreads();
  return t;
}

// Generic row kernel: thread owns column vectors jv = q*NT + tid (q < CPT), V columns each.
template <typename T, int V, int CPT, int KU>
__global__ void __launch_bounds__(256) k_rows_ldg(RowParams p) {
  using VT = typename VecL<T, V>::type;
  using Acc = T;                         // fp32 k-sums for fp32 data, fp64 for fp64 data
  __shared__ double sh[32];
  const int NT = blockDim.x;
  const int64_t m = p.m, mv = m / V;
  const T* C = static_cast<const T*>(p.C);
  const T* G = static_cast<const T*>(p.G);
  for (int64_t u = blockIdx.x; u < p.U; u += gridDim.x) {
    const int64_t b = u / p.upp, cu = u - b * p.upp;
    if (!p.state[b].active) continue;    // block-uniform
    const int64_t i0 = cu * p.rpu;
    const int64_t i1 = min(p.R, i0 + p.rpu);
    const double inv_eps = 1.0 / p.eps[b];
    const float c2 = (float)(COT_LOG2E * inv_eps);
    double z[CPT][V], P[CPT][V];
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      const int64_t jv = (int64_t)q * NT + threadIdx.x;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        P[q][v] = 0.0;
        z[q][v] = jv < mv ? p.z_hat[b * m + jv * V + v] : 0.0;
      }
    }
    for (int64_t i = i0; i < i1; ++i) {
      const VT* Grow = reinterpret_cast<const VT*>(G + (b * p.R + i) * m);
      const VT* Crow = reinterpret_cast<const VT*>(C + (b * p.n * p.R + i) * m);
      const int64_t kstride = p.R * mv;   // vectors between consecutive blocks k
      T g[CPT][V];
      Acc s[CPT][V];
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const int64_t jv = (int64_t)q * NT + threadIdx.x;
        VT gv = jv < mv ? Grow[jv] : VT{};
        VecL<T, V>::unpack(gv, g[q]);
#pragma unroll
        for (int v = 0; v < V; ++v) s[q][v] = Acc(0);
      }
      // ---- streamed k-sum: the n*m^2 Gibbs-kernel evaluations of this iteration
      int64_t k = 0;
      if (p.pre) {   // NEXT-1 (Alg. 2 line 1 as written): s_ij was computed once by cerot_precompute
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
          const int64_t jv = (int64_t)q * NT + threadIdx.x;
          VT cvv = jv < mv ? __ldg(Crow + jv) : VT{};
          T c[V];
          VecL<T, V>::unpack(cvv, c);
#pragma unroll
          for (int v = 0; v < V; ++v) s[q][v] = c[v];
        }
        k = p.n;
      }
      for (; k + KU <= p.n; k += KU) {
        VT cv[KU][CPT];
#pragma unroll
        for (int uu = 0; uu < KU; ++uu)
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            const int64_t jv = (int64_t)q * NT + threadIdx.x;
            cv[uu][q] = jv < mv ? __ldcs(Crow + (k + uu) * kstride + jv) : VT{};
          }
#pragma unroll
        for (int uu = 0; uu < KU; ++uu)
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            T c[V];
            VecL<T, V>::unpack(cv[uu][q], c);
#pragma unroll
            for (int v = 0; v < V; ++v) {
              if constexpr (sizeof(T) == 4)
                s[q][v] += ex2((g[q][v] - c[v]) * c2);
              else
                s[q][v] += exp((g[q][v] - c[v]) * inv_eps);
            }
          }
      }
      for (; k < p.n; ++k) {
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
          const int64_t jv = (int64_t)q * NT + threadIdx.x;
          VT cvv = jv < mv ? __ldcs(Crow + k * kstride + jv) : VT{};
          T c[V];
          VecL<T, V>::unpack(cvv, c);
#pragma unroll
          for (int v = 0; v < V; ++v) {
            if constexpr (sizeof(T) == 4)
              s[q][v] += ex2((g[q][v] - c[v]) * c2);
            else
              s[q][v] += exp((g[q][v] - c[v]) * inv_eps);
          }
        }
      }
      // ---- row epilogue (fp64): M_i, r_i, w_hat_i, column partials
      double x[CPT][V];
      double lmax = -INFINITY;
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const bool ok = (int64_t)q * NT + threadIdx.x < mv;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          x[q][v] = ok ? z[q][v] - (double)g[q][v] * inv_eps : -INFINITY;
          lmax = fmax(lmax, x[q][v]);
        }
      }
      const double M = blk_max(lmax, sh);
      double t[CPT][V];
      double lsum = 0.0;
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const bool ok = (int64_t)q * NT + threadIdx.x < mv;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          double e;
          if constexpr (sizeof(T) == 4)
            e = (double)ex2((float)((x[q][v] - M) * COT_LOG2E));
          else
            e = exp(x[q][v] - M);
          t[q][v] = ok ? (double)s[q][v] * e : 0.0;
          lsum += t[q][v];
        }
      }
      const double r = blk_sum(lsum, sh);
      const double a = p.alpha[b * m + p.row_begin + i];
      if (threadIdx.x == 0) p.w_hat[b * m + p.row_begin + i] = log(a) - M - log(r);
      const double rho = a / r;
#pragma unroll
      for (int q = 0; q < CPT; ++q)
#pragma unroll
        for (int v = 0; v < V; ++v) P[q][v] = fma(rho, t[q][v], P[q][v]);
    }
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      const int64_t jv = (int64_t)q * NT + threadIdx.x;
      if (jv < mv) {
#pragma unroll
        for (int v = 0; v < V; ++v) p.partials[u * m + jv * V + v] = P[q][v];
      }
    }
  }
}

// Column pass. grid = (ceil(m/32), B), 256 threads = 8 warps; lane <-> column, warp w sums the units
// w, w+8, ... in order, then warp 0 combines the 8 warp sums in order: a fixed summation tree.
__global__ void __launch_bounds__(256) k_cols(const double* __restrict__ partials, int64_t upp, int64_t m,
                                              int64_t n, const double* __restrict__ beta, double* __restrict__ z_hat,
                                              double* __restrict__ resid_part, SolverState* __restrict__ state,
                                              unsigned* __restrict__ counters, double tol, int64_t check_every) {
  const int64_t b = blockIdx.y;
  const int ntiles = gridDim.x;
  if (!state[b].active) return;          // block-uniform; only the last block of this launch changes it
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  __shared__ double sh[8][33];
  __shared__ bool is_last;
  double acc = 0.0;
  if (j < m)
    for (int64_t c = w; c < upp; c += 8) acc += __ldcg(partials + (b * upp + c) * m + j);
  sh[w][lane] = acc;
  __syncthreads();
  if (w == 0) {
    double cj = 0.0;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) cj += sh[ww][lane];
    double dev = 0.0;
    bool uf = false;
    if (j < m) {
      const double bj = beta[b * m + j];
      dev = fabs(cj - bj);
      uf = !(cj >= 1e-28);               // also catches NaN
      z_hat[b * m + j] += log(bj) - log(cj);
    }
    dev = warp_sum(dev);
    if (__any_sync(0xffffffffu, uf) && lane == 0) atomicOr(&state[b].flags, (int)STATE_UNDERFLOW);
    if (lane == 0) resid_part[b * ntiles + blockIdx.x] = dev;
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

// Validation of alpha, beta (entries > 0; sums equal to 1e-6 relative) + state reset +
// optional cold start z_hat = 0 (q = 1_m, Alg. 2 line 2). One block per problem.
__global__ void __launch_bounds__(256) k_init(const double* __restrict__ alpha, const double* __restrict__ beta,
                                              int64_t m, uint32_t flags, double* __restrict__ z_hat,
                                              SolverState* __restrict__ state, unsigned* __restrict__ counters,
                                              unsigned* __restrict__ grid_bar) {
  __shared__ double sh[32];
  const int64_t b = blockIdx.x;
  if (b == 0 && threadIdx.x == 0) {
    grid_bar[0] = 0u;
    grid_bar[1] = 0u;
    grid_bar[2] = 0u;
    grid_bar[3] = 0u;
  }
  double sa = 0.0, sb = 0.0, bad = 0.0;
  for (int64_t j = threadIdx.x; j < m; j += blockDim.x) {
    const double a = alpha[b * m + j], bb = beta[b * m + j];
    sa += a;
    sb += bb;
    bad += (!(a > 0.0) || !(bb > 0.0) || !finite_f(a) || !finite_f(bb)) ? 1.0 : 0.0;
    if (flags & COT_COLD_START) z_hat[b * m + j] = 0.0;
  }
  sa = blk_sum(sa, sh);
  sb = blk_sum(sb, sh);
  bad = blk_sum(bad, sh);
  if (threadIdx.x == 0) {
    const bool mism = fabs(sa - sb) > 1e-6 * fmax(fabs(sa), fabs(sb));
    SolverState st;
    st.iters = 0;
    st.converged = 0;
    st.residual = INFINITY;
    st.flags = (bad > 0.0 || mism) ? STATE_BAD_MARGINAL : 0;
    st.active = st.flags ? 0 : 1;
    if (!(sa < kDetAlphaMax)) st.flags |= STATE_DET_RANGE;
    st.pad = 0;
    state[b] = st;
    counters[b] = 0u;
  }
}

// ------------------------------------------------------------------------------------ launchers
cudaError_t launch_init(const double* alpha, const double* beta, int64_t B, int64_t m, uint32_t flags, double* z_hat,
                        const Workspace& ws, cudaStream_t s) {
  // the persistent kernels' device-wide state (LL lines, K-ITER-RES sums and counters) starts from zero on every
  // (re)initialisation of the workspace
  if (ws.ll_base) {
    const cudaError_t e = cudaMemsetAsync(ws.ll_base, 0, ws.ll_bytes, s);
    if (e != cudaSuccess) return e;
  }
  k_init<<<(unsigned)B, 256, 0, s>>>(alpha, beta, m, flags, z_hat, ws.state, ws.counters, ws.grid_bar);
  return cudaGetLastError();
}

template <typename T, int V>
static cudaError_t rows_dispatch(const RowParams& rp, int grid, int64_t m, cudaStream_t s) {
  const int64_t mv = m / V;
  int nt = (int)((mv + 31) / 32 * 32);
  if (nt > 256) nt = 256;
  const int64_t cpt = (mv + nt - 1) / nt;
  constexpr int KU = sizeof(T) == 4 ? 8 : 4;
  if (cpt <= 1)
    k_rows_ldg<T, V, 1, KU><<<grid, nt, 0, s>>>(rp);
  else if (cpt <= 2)
    k_rows_ldg<T, V, 2, KU><<<grid, nt, 0, s>>>(rp);
  else if (cpt <= 4)
    k_rows_ldg<T, V, 4, KU><<<grid, nt, 0, s>>>(rp);
  else if (cpt <= 8)
    k_rows_ldg<T, V, 8, KU><<<grid, nt, 0, s>>>(rp);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_rows(const IterArgs& a, const Workspace& ws, const UnitPlan& up, int parity, cudaStream_t s) {
  RowParams rp;
  rp.C = a.C;
  rp.G = a.G;
  rp.alpha = a.alpha;
  rp.z_hat = a.z_hat;
  rp.w_hat = a.w_hat;
  rp.eps = a.eps;
  rp.n = a.n;
  rp.m = a.m;
  rp.R = a.R;
  rp.row_begin = a.row_begin;
  rp.rpu = up.rpu;
  rp.upp = up.upp;
  rp.U = up.U;
  rp.partials = ws.partials[parity];
  rp.state = ws.state;
  rp.pre = (a.flags & COT_PRECOMPUTED) ? 1 : 0;
  if (a.dtype == COT_F32) {
    if (a.m % 4 == 0) return rows_dispatch<float, 4>(rp, up.grid, a.m, s);
    return rows_dispatch<float, 1>(rp, up.grid, a.m, s);
  }
  if (a.m % 2 == 0) return rows_dispatch<double, 2>(rp, up.grid, a.m, s);
  return rows_dispatch<double, 1>(rp, up.grid, a.m, s);
}

// The condition of cerot_solve's device-side loop: continue while some problem is still active and fewer than
// max_iter iterations have been launched (one block).
__global__ void __launch_bounds__(256) k_loop_cond(cudaGraphConditionalHandle h, const SolverState* __restrict__ state,
                                                   int64_t B, unsigned* __restrict__ ctr, int64_t max_iter) {
  int any = 0;
  for (int64_t b = threadIdx.x; b < B; b += blockDim.x) any |= state[b].active;
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) {
    const unsigned done = ctr[0] + 1u;
    ctr[0] = done;
    cudaGraphSetConditional(h, (any && (int64_t)done < max_iter) ? 1u : 0u);
  }
}

cudaError_t launch_ldg_loop(const IterArgs& a, const Workspace& ws, const UnitPlan& up, int64_t max_iter,
                            cudaStream_t s) {
  if (max_iter < 1) return cudaSuccess;
  cudaGraph_t g = nullptr, body = nullptr;
  cudaGraphExec_t ge = nullptr;
  cudaError_t e = cudaGraphCreate(&g, 0);
  if (e != cudaSuccess) return e;
  cudaGraphConditionalHandle h;
  e = cudaGraphConditionalHandleCreate(&h, g, 1u, cudaGraphCondAssignDefault);
  cudaGraphNode_t node;
  cudaGraphNodeParams cp = {};
  if (e == cudaSuccess) {
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    e = cudaGraphAddNode(&node, g, nullptr, 0, &cp);
  }
  cudaStream_t cs = nullptr;
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  if (e == cudaSuccess) {   // the loop body: one iteration of every active problem, then the condition
    body = cp.conditional.phGraph_out[0];
    e = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
    if (e == cudaSuccess) {
      cudaError_t e1 = launch_rows(a, ws, up, 0, cs);
      if (e1 == cudaSuccess) e1 = launch_cols(a, ws, up, 0, cs);
      if (e1 == cudaSuccess) {
        k_loop_cond<<<1, 256, 0, cs>>>(h, ws.state, a.B, ws.loopctl, max_iter);
        e1 = cudaGetLastError();
      }
      e = cudaStreamEndCapture(cs, &body);
      if (e1 != cudaSuccess) e = e1;
    }
  }
  if (e == cudaSuccess) e = cudaGraphInstantiate(&ge, g, 0);
  if (e == cudaSuccess) e = cudaMemsetAsync(ws.loopctl, 0, 16, s);
  if (e == cudaSuccess) e = cudaGraphLaunch(ge, s);
  if (ge) cudaGraphExecDestroy(ge);   // freed once the in-flight launch completes
  if (g) cudaGraphDestroy(g);
  if (cs) cudaStreamDestroy(cs);
  return e;
}

cudaError_t launch_cols(const IterArgs& a, const Workspace& ws, const UnitPlan& up, int parity, cudaStream_t s) {
  dim3 grid((unsigned)((a.m + 31) / 32), (unsigned)a.B);
  k_cols<<<grid, 256, 0, s>>>(ws.partials[parity], up.upp, a.m, a.n, a.beta, a.z_hat, ws.resid_part, ws.state,
                              ws.counters, a.tol, a.check_every > 0 ? a.check_every : 1);
  return cudaGetLastError();
}

}  // namespace cot
