// Kernels of the row-sharded path: GPU g holds rows [row_begin, row_begin + R) of every
// block. The p-update of those rows is local; the column sums c_j = sum_i (alpha_i / r_i) t_ij are partial
// per GPU and are summed across GPUs (ncclAllReduce, one m-length fp64 vector per iteration), after which
// every GPU applies the identical q-update z_hat_j += log beta_j - log c_j and monitor. The plan
// reductions follow the same pattern: local partials -> one allreduce -> identical report on every GPU.
// With one GPU (no communicator) these kernels give the unsharded results; cerot_plan uses them too.
#include "common.cuh"
#include "internal.h"

namespace cot {

// c[b][j] = sum_u partials[b*upp + u][j], units in a fixed order (the same tree as k_cols: warp w sums
// units w, w+8, ...; warp 0 combines the 8 warp sums in order). grid = (ceil(m/32), B), 256 threads.
__global__ void __launch_bounds__(256) k_colsum(const double* __restrict__ partials, int64_t upp, int64_t m,
                                                const SolverState* __restrict__ state, double* __restrict__ c) {
  const int64_t b = blockIdx.y;
  if (state && !state[b].active) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  __shared__ double sh[8][33];
  double acc = 0.0;
  if (j < m) {
    // units w, w + 8, ... in order; eight loads in flight per step (one L2 latency per eight units, not one each)
    const double* pc = partials + b * upp * m + j;
    int64_t u = w;
    for (; u + 56 < upp; u += 64) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = __ldcg(pc + (u + 8 * q) * m);
#pragma unroll
      for (int q = 0; q < 8; ++q) acc += v[q];
    }
    for (; u < upp; u += 8) acc += __ldcg(pc + u * m);
  }
  sh[w][lane] = acc;
  __syncthreads();
  if (w == 0 && j < m) {
    double cj = 0.0;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) cj += sh[ww][lane];
    c[b * m + j] = cj;
  }
}

// q-update from the (reduced) column sums: z_hat_j += log beta_j - log c_j, monitor n * sum_j |c_j - beta_j|
// with a last-block-done reduction in a fixed order, iteration count and freeze rule.
__global__ void __launch_bounds__(256) k_zupdate(const double* __restrict__ c, int64_t m, int64_t n,
                                                 const double* __restrict__ beta, double* __restrict__ z_hat,
                                                 double* __restrict__ resid_part, SolverState* __restrict__ state,
                                                 unsigned* __restrict__ counters, double tol, int64_t check_every) {
  const int64_t b = blockIdx.y;
  const int ntiles = gridDim.x;
  if (!state[b].active) return;
  const int lane = threadIdx.x & 31;
  __shared__ bool is_last;
  if (threadIdx.x < 32) {
    const int64_t j = (int64_t)blockIdx.x * 32 + lane;
    double dev = 0.0;
    bool uf = false;
    if (j < m) {
      const double cj = c[b * m + j];
      const double bj = beta[b * m + j];
      dev = fabs(cj - bj);
      uf = !(cj >= 1e-28);
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
  if (is_last) {
    __threadfence();
    // the tiles' partial residuals summed in tile order by thread 0, read by the whole warp first (one L2
    // latency per 32 tiles instead of one per tile)
    __shared__ double rp[32];
    double r = 0.0;
    for (int t0 = 0; t0 < ntiles; t0 += 32) {
      const int nt = min(32, ntiles - t0);
      if (lane < nt) rp[lane] = __ldcg(resid_part + b * ntiles + t0 + lane);
      __syncwarp();
      if (threadIdx.x == 0)
        for (int t = 0; t < nt; ++t) r += rp[t];
      __syncwarp();
    }
    if (threadIdx.x == 0) {
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
}

// Local plan reductions into buf[b] = {transport, entropy sum, sum_i |r_i - alpha_i|, mass,
// sum_{held rows} w_hat_i alpha_i, c_0 .. c_{m-1}} (all over the rows this call holds).
// grid = (ceil(m/32), B), 256 threads: block x sums its 32 columns over the units (warp w takes units w, w+8,
// ..., lanes the columns; the 8 warp sums combined in order, as k_colsum); block 0 also forms the scalars.
__global__ void __launch_bounds__(256) k_plan_reduce_local(const double* __restrict__ partials,
                                                           const double* __restrict__ scal, int64_t upp, int64_t m,
                                                           int64_t row_begin, int64_t R,
                                                           const double* __restrict__ alpha,
                                                           const double* __restrict__ w_hat, double* __restrict__ buf) {
  __shared__ double sh[32];
  __shared__ double shc[8][33];
  const int64_t b = blockIdx.y;
  double* o = buf + b * (kPlanBufHead + m);
  {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t j = (int64_t)blockIdx.x * 32 + lane;
    double acc = 0.0;
    if (j < m)
      for (int64_t u = w; u < upp; u += 8) acc += partials[(b * upp + u) * m + j];
    shc[w][lane] = acc;
    __syncthreads();
    if (w == 0 && j < m) {
      double c = 0.0;
#pragma unroll
      for (int ww = 0; ww < 8; ++ww) c += shc[ww][lane];
      o[kPlanBufHead + j] = c;
    }
  }
  if (blockIdx.x != 0) return;
  double dot = 0.0;
  for (int64_t i = threadIdx.x; i < R; i += blockDim.x) dot += w_hat[b * m + row_begin + i] * alpha[b * m + row_begin + i];
  dot = warp_sum(dot);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sh[wid] = dot;
  __syncthreads();
  if (threadIdx.x == 0) {
    double d = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) d += sh[w];
    double tr = 0.0, en = 0.0, rl1 = 0.0, mass = 0.0;
    for (int64_t u = 0; u < upp; ++u) {
      const double* sc = scal + (b * upp + u) * kPlanScalars;
      tr += sc[0];
      en += sc[1];
      rl1 += sc[2];
      mass += sc[3];
    }
    o[0] = tr;
    o[1] = en;
    o[2] = rl1;
    o[3] = mass;
    o[4] = d;
  }
}

// The report (cot_report field order) from the reduced buffer; identical on every GPU.
__global__ void __launch_bounds__(256) k_plan_finalize_buf(const double* __restrict__ buf, int64_t m, int64_t n,
                                                           const double* __restrict__ beta,
                                                           const double* __restrict__ z_hat,
                                                           const double* __restrict__ eps,
                                                           const SolverState* __restrict__ state,
                                                           double* __restrict__ report) {
  __shared__ double sh[3][32];
  const int64_t b = blockIdx.x;
  const double* o = buf + b * (kPlanBufHead + m);
  double cl1 = 0.0, cl2 = 0.0, dz = 0.0;
  for (int64_t j = threadIdx.x; j < m; j += blockDim.x) {
    const double dv = o[kPlanBufHead + j] - beta[b * m + j];
    cl1 += fabs(dv);
    cl2 += dv * dv;
    dz += z_hat[b * m + j] * beta[b * m + j];
  }
  cl1 = warp_sum(cl1);
  cl2 = warp_sum(cl2);
  dz = warp_sum(dz);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    sh[0][wid] = cl1;
    sh[1][wid] = cl2;
    sh[2][wid] = dz;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a1 += sh[0][w];
      a2 += sh[1][w];
      a3 += sh[2][w];
    }
    const double nn = (double)n, e = eps[b];
    const double tr = o[0], en = o[1], rl1 = o[2], mass = o[3], dw = o[4];
    double* rep = report + b * kReportDoubles;
    rep[0] = nn * tr;                       // objective: transport cost of the full plan
    rep[1] = nn * (tr + e * en);            // regularised primal
    rep[2] = nn * e * (dw + a3 - mass);     // dual (phi*(y) = eps e^{y/eps})
    rep[3] = nn * rl1;                      // ||T 1 - a||_1
    rep[4] = nn * a1;                       // ||T^T 1 - b||_1
    rep[5] = sqrt(nn * a2);                 // ||T^T 1 - b||_2
    rep[6] = nn * mass;                     // full plan mass
    rep[7] = state ? state[b].residual : 0.0;
  }
}

cudaError_t launch_colsum(const Workspace& ws, const UnitPlan& up, int64_t B, int64_t m, int parity, double* c,
                          cudaStream_t s) {
  dim3 grid((unsigned)((m + 31) / 32), (unsigned)B);
  k_colsum<<<grid, 256, 0, s>>>(ws.partials[parity], up.upp, m, ws.state, c);
  return cudaGetLastError();
}

cudaError_t launch_zupdate(const double* c, const double* beta, int64_t B, int64_t m, int64_t n, double tol,
                           int64_t check_every, double* z_hat, const Workspace& ws, cudaStream_t s) {
  dim3 grid((unsigned)((m + 31) / 32), (unsigned)B);
  k_zupdate<<<grid, 32, 0, s>>>(c, m, n, beta, z_hat, ws.resid_part, ws.state, ws.counters, tol,
                                check_every > 0 ? check_every : 1);
  return cudaGetLastError();
}

cudaError_t launch_plan_reduce_local(const IterArgs& a, const Workspace& ws, const UnitPlan& up, double* buf,
                                     cudaStream_t s) {
  dim3 grid((unsigned)((a.m + 31) / 32), (unsigned)a.B);
  k_plan_reduce_local<<<grid, 256, 0, s>>>(ws.partials[0], ws.plan_scal, up.upp, a.m, a.row_begin, a.R, a.alpha,
                                           a.w_hat, buf);
  return cudaGetLastError();
}

cudaError_t launch_plan_finalize_buf(const IterArgs& a, const Workspace& ws, const double* buf, double* report,
                                     cudaStream_t s) {
  k_plan_finalize_buf<<<(unsigned)a.B, 256, 0, s>>>(buf, a.m, a.n, a.beta, a.z_hat, a.eps, ws.state, report);
  return cudaGetLastError();
}

}  // namespace cot
