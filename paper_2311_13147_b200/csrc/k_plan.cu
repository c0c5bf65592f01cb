// K-PLAN: plan reconstruction T_ijk = exp(w_hat_i + z_hat_j - C_ijk/eps) (Alg. 2 lines 7-9, P:434-436;
// eq. optimality_condition) fused with the fp64 reductions of the report:
//   transport sum C T, entropy sum T (log T - 1), row sums r_i (-> row residual, mass), column sums c_j.
// Numerics: y_ij = w_hat_i + z_hat_j - G_ij/eps and E_ij = exp(y_ij) in fp64 once per (i,j);
// a_ijk = (G_ij - C_ijk)/eps <= 0 in fp64, exp(a) in fp32 (accurate exp2f, not ex2.approx),
// T = E * exp(a) and log T = y + a in fp64. All sums fp64 in a fixed order (deterministic).
#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace cot {

template <typename T, int V>
struct VecP;
template <>
struct VecP<float, 4> {
  using type = float4;
  __device__ static void unpack(const type& v, float* o) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
  __device__ static type pack(const float* o) { return make_float4(o[0], o[1], o[2], o[3]); }
};
template <>
struct VecP<float, 1> {
  using type = float;
  __device__ static void unpack(const type& v, float* o) { o[0] = v; }
  __device__ static type pack(const float* o) { return o[0]; }
};
template <>
struct VecP<double, 2> {
  using type = double2;
  __device__ static void unpack(const type& v, double* o) { o[0] = v.x; o[1] = v.y; }
  __device__ static type pack(const double* o) { return make_double2(o[0], o[1]); }
};
template <>
struct VecP<double, 1> {
  using type = double;
  __device__ static void unpack(const type& v, double* o) { o[0] = v; }
  __device__ static type pack(const double* o) { return o[0]; }
};

struct PlanParams {
  const void* C;
  const void* G;
  const double* alpha;
  const double* w_hat;
  const double* z_hat;
  const double* eps;
  void* T;               // [B][n][R][m] or nullptr
  int64_t n, m, R, row_begin, rpu, upp, U;
  double* partials;      // [U][m] column partials
  double* scal;          // [U][kPlanScalars]
  const SolverState* state;
};

__device__ __forceinline__ double pblk_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < nw; ++w) t += sh[w];
  __syncthreads();
  return t;
}

template <typename T, int V, int CPT>
__global__ void __launch_bounds__(256) k_plan(PlanParams p) {
  using VT = typename VecP<T, V>::type;
  __shared__ double sh[32];
  const int NT = blockDim.x;
  const int64_t m = p.m, mv = m / V;
  const T* C = static_cast<const T*>(p.C);
  const T* G = static_cast<const T*>(p.G);
  T* Tout = static_cast<T*>(p.T);
  for (int64_t u = blockIdx.x; u < p.U; u += gridDim.x) {
    const int64_t b = u / p.upp, cu = u - b * p.upp;
    const int64_t i0 = cu * p.rpu;
    const int64_t i1 = min(p.R, i0 + p.rpu);
    const double eps = p.eps[b];
    const double inv_eps = 1.0 / eps;
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
    double transport = 0.0, ent = 0.0, rl1 = 0.0, mass = 0.0;
    for (int64_t i = i0; i < i1; ++i) {
      const int64_t gi = p.row_begin + i;
      const double wi = p.w_hat[b * m + gi];
      const VT* Grow = reinterpret_cast<const VT*>(G + (b * p.R + i) * m);
      const VT* Crow = reinterpret_cast<const VT*>(C + (b * p.n * p.R + i) * m);
      VT* Trow = Tout ? reinterpret_cast<VT*>(Tout + (b * p.n * p.R + i) * m) : nullptr;
      const int64_t kstride = p.R * mv;
      T g[CPT][V];
      double y[CPT][V], E[CPT][V];
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const int64_t jv = (int64_t)q * NT + threadIdx.x;
        VT gv = jv < mv ? Grow[jv] : VT{};
        VecP<T, V>::unpack(gv, g[q]);
#pragma unroll
        for (int v = 0; v < V; ++v) {
          y[q][v] = wi + z[q][v] - (double)g[q][v] * inv_eps;
          E[q][v] = exp(y[q][v]);
        }
      }
      double row = 0.0;
      // blocks in groups of KU: the KU loads of a group are issued before any arithmetic (memory parallelism:
      // 16 vectors per thread in flight, 64 KB per 256-thread CTA; the sums still run in k order, so the grouping
      // does not change a bit. C4: KU = 4 left k_plan at 0.44 of HBM, 186 us for its 537 MB)
      constexpr int KU = CPT >= 8 ? 2 : 16 / CPT;
      auto element = [&](int q, const VT& cvv, T* tout) {
        T c[V];
        VecP<T, V>::unpack(cvv, c);
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const double a = ((double)g[q][v] - (double)c[v]) * inv_eps;   // <= 0
          double e;
          if constexpr (sizeof(T) == 4)
            e = (double)exp2f((float)(a * COT_LOG2E));
          else
            e = exp(a);
          const double Tv = E[q][v] * e;
          transport = fma((double)c[v], Tv, transport);
          ent = fma(Tv, (y[q][v] + a) - 1.0, ent);
          row += Tv;
          P[q][v] += Tv;
          tout[v] = (T)Tv;
        }
      };
      int64_t k = 0;
      for (; k + KU <= p.n; k += KU) {
        VT cv[KU][CPT];
#pragma unroll
        for (int kk = 0; kk < KU; ++kk)
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            const int64_t jv = (int64_t)q * NT + threadIdx.x;
            if (jv < mv) cv[kk][q] = __ldcs(Crow + (k + kk) * kstride + jv);
          }
#pragma unroll
        for (int kk = 0; kk < KU; ++kk)
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            const int64_t jv = (int64_t)q * NT + threadIdx.x;
            if (jv >= mv) continue;
            T tout[V];
            element(q, cv[kk][q], tout);
            if (Trow) __stcs(Trow + (k + kk) * kstride + jv, VecP<T, V>::pack(tout));
          }
      }
      for (; k < p.n; ++k) {
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
          const int64_t jv = (int64_t)q * NT + threadIdx.x;
          if (jv >= mv) continue;
          T tout[V];
          element(q, __ldcs(Crow + k * kstride + jv), tout);
          if (Trow) __stcs(Trow + k * kstride + jv, VecP<T, V>::pack(tout));
        }
      }
      const double r = pblk_sum(row, sh);
      rl1 += fabs(r - p.alpha[b * m + gi]);
      mass += r;
    }
    transport = pblk_sum(transport, sh);
    ent = pblk_sum(ent, sh);
    if (threadIdx.x == 0) {
      double* sc = p.scal + u * kPlanScalars;
      sc[0] = transport;
      sc[1] = ent;
      sc[2] = rl1;
      sc[3] = mass;
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

template <typename T, int V>
static cudaError_t plan_dispatch(const PlanParams& pp, int grid, int64_t m, cudaStream_t s) {
  const int64_t mv = m / V;
  int nt = (int)((mv + 31) / 32 * 32);
  if (nt > 256) nt = 256;
  const int64_t cpt = (mv + nt - 1) / nt;
  if (cpt <= 1)
    k_plan<T, V, 1><<<grid, nt, 0, s>>>(pp);
  else if (cpt <= 2)
    k_plan<T, V, 2><<<grid, nt, 0, s>>>(pp);
  else if (cpt <= 4)
    k_plan<T, V, 4><<<grid, nt, 0, s>>>(pp);
  else if (cpt <= 8)
    k_plan<T, V, 8><<<grid, nt, 0, s>>>(pp);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_plan(const IterArgs& a, const Workspace& ws, const UnitPlan& up, void* T_blocks, cudaStream_t s) {
  PlanParams pp;
  pp.C = a.C;
  pp.G = a.G;
  pp.alpha = a.alpha;
  pp.w_hat = a.w_hat;
  pp.z_hat = a.z_hat;
  pp.eps = a.eps;
  pp.T = T_blocks;
  pp.n = a.n;
  pp.m = a.m;
  pp.R = a.R;
  pp.row_begin = a.row_begin;
  pp.rpu = up.rpu;
  pp.upp = up.upp;
  pp.U = up.U;
  pp.partials = ws.partials[0];
  pp.scal = ws.plan_scal;
  pp.state = ws.state;
  // a unit's CTA has one thread per vector of columns (32 for m = 128): with small m, keep up to 32 such CTAs
  // resident per SM (C5: 4096 single-warp units; 4 per SM left the T-block stream at 1.5 TB/s)
  const int64_t vw = a.dtype == COT_F32 ? (a.m % 4 == 0 ? 4 : 1) : (a.m % 2 == 0 ? 2 : 1);
  const int64_t nt = std::min<int64_t>(256, (a.m / vw + 31) / 32 * 32);
  const int per_sm = (int)std::max<int64_t>(4, std::min<int64_t>(32, 1024 / nt));
  const int grid = (int)std::min<int64_t>(up.U, (int64_t)device_sm_count() * per_sm);
  cudaError_t e;
  if (a.dtype == COT_F32)
    e = (a.m % 4 == 0) ? plan_dispatch<float, 4>(pp, grid, a.m, s) : plan_dispatch<float, 1>(pp, grid, a.m, s);
  else
    e = (a.m % 2 == 0) ? plan_dispatch<double, 2>(pp, grid, a.m, s) : plan_dispatch<double, 1>(pp, grid, a.m, s);
  return e;
}

}  // namespace cot
