// K-BATCH: cluster-resident cyclic Sinkhorn for small problems (C5: B = 4096 x (n = 16, m = 128); C2), the
// same arithmetic as k_rows_ldg + k_cols (k_iter.cu) with the whole problem on chip for all iterations.
//
// One thread-block cluster of NCL = 8 CTAs per problem. CTA c holds rows [c*RB, (c+1)*RB) of every cost
// block in shared memory (RB*n*m fp32; 128 KiB for C5), loaded once with TMA bulk copies, plus its G rows
// and a replica of z_hat. One warp per row, VEC = 4 columns per lane (x VPL):
//   k-sum       s'_ij = sum_k exp2(a_ij - C_ijk log2e/eps) from shared memory (FFMA + MUFU.EX2 + FADD), with
//               the integer shift a_ij = round(G_ij log2e/eps) (s'_ij in [0.7, 1.42 n]);
//   epilogue    t_ij = s'_ij 2^{kz_j - a_ij - kM_i} Fz_j with z_hat_j log2e = kz_j + log2 Fz_j split once per
//               column per iteration (kept in the replica next to z_hat) and kM_i = max_j (kz_j - a_ij) by one
//               integer warp reduction: the exponent goes into the fp64 bits, one fp64 product, no MUFU and
//               no conversion per element. r_i by warp shuffles (no block barrier: a row lives in one warp),
//               w_hat_i = log alpha_i - kM_i ln2 - log r_i, column terms (alpha_i / r_i) t_ij in fp64;
//   columns     per-CTA column partials in shared memory; after a cluster barrier CTA c sums the 8 CTAs'
//               partials of its column slice through DSMEM in CTA order (deterministic), applies the
//               q-update z_hat_j += log beta_j - log c_j and writes z_hat_j into every CTA's replica (DSMEM);
//               a second cluster barrier publishes the new z_hat. The monitor n*sum|c_j - beta_j| is combined
//               through CTA 0's shared memory and read by all CTAs (uniform freeze decision).
// No HBM traffic per iteration: the bound is the SFU (n*m^2 MUFU.EX2 per iteration per problem) plus two
// cluster barriers.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace cot {

constexpr int kMaxNCL = 16;   // CTAs per cluster: up to the non-portable maximum

struct BatchParams {
  const float* C;        // [B][n][m][m]
  const float* G;        // [B][m][m]
  const double* alpha;   // [B][m]
  const double* beta;    // [B][m]
  double* w_hat;         // [B][m]
  double* z_hat;         // [B][m]
  const double* eps;     // [B]
  SolverState* state;    // [B]
  int n, m, RB;          // rows per CTA
  int iters;
  double tol;
  long long check_every;
  int pre;               // precomputed mode (NEXT-1): C is S [B][1][m][m], s_ij = S_ij
  int ncl;               // CTAs per cluster (one problem per cluster)
  int ne;                // warp-specialised kernel: epilogue warps (the rest of the block: k-sum warps)
  int gs_log;            // log2 of the column-pass group (a power of two >= ncl: 8 or 16 lanes)
  unsigned long long* trace;   // diagnostics (COT_TRACE=1): [grid][8] cycle counters, or nullptr
};

template <int VPL, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_batch_cluster(BatchParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const int ncl = p.ncl;
  const int64_t b = blockIdx.x / ncl;                       // problem of this cluster
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int n = p.n, m = p.m, RB = p.RB, mv = m >> 2;
  const int r0 = crank * RB;                                // first row of this CTA
  const int nrows = max(0, min(RB, m - r0));
  // ---- shared memory: C rows [RB][n][m] f32 | G rows [RB][m] f32, then the shifts a_ij (int32) in place |
  //      z [m] f64 | Fz [m] f64 | kz [m] i32 | warp partials [nw][m] f64 | CTA partial [m] f64 | monitor
  //      partials [NCL] f64 | row stats | beta | mbarrier
  float* Cs = reinterpret_cast<float*>(smem);
  float* Gs = Cs + (size_t)RB * n * m;
  int* As = reinterpret_cast<int*>(Gs);
  double* zs = reinterpret_cast<double*>(Gs + (size_t)RB * m);
  double* zf = zs + m;
  int* zk = reinterpret_cast<int*>(zf + m);
  double* wpart = reinterpret_cast<double*>(zk + m);   // m % 4 == 0: 8-byte aligned
  double* cpart = wpart + (size_t)nwarps * m;
  double* mon = cpart + m;
  double* rstat = mon + kMaxNCL;                                // [RB][4]: M_i, r_i, alpha_i, log alpha_i
  double* bcol = rstat + (size_t)RB * 4;                     // [m][2]: beta_j, log beta_j
  uint64_t* bar = reinterpret_cast<uint64_t*>(bcol + (size_t)m * 2);
  __shared__ int s_flags;

  SolverState st = p.state[b];
  if (!st.active) return;                                   // cluster-uniform
  const double inv_eps = 1.0 / p.eps[b];
  const float c2 = (float)(COT_LOG2E * inv_eps);

  // ---- load this CTA's rows of C (all n blocks) and G once (TMA bulk copies, one mbarrier)
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    s_flags = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0 && nrows > 0) {
    const uint32_t row_bytes = (uint32_t)m * 4u;
    mbar_arrive_expect_tx(bar, (uint32_t)nrows * (uint32_t)(n + 1) * row_bytes);
    const uint64_t pol = policy_evict_first();
    for (int i = 0; i < nrows; ++i) {
      for (int k = 0; k < n; ++k)
        bulk_g2s(Cs + ((size_t)i * n + k) * m, p.C + (((size_t)b * n + k) * m + r0 + i) * m, row_bytes, bar, pol);
      bulk_g2s(Gs + (size_t)i * m, p.G + ((size_t)b * m + r0 + i) * m, row_bytes, bar, pol);
    }
  }
  for (int j = threadIdx.x; j < m; j += blockDim.x) {
    zs[j] = p.z_hat[b * m + j];
    zf[j] = split_z(zs[j], zk[j]);
    const double bj = p.beta[b * m + j];
    bcol[2 * j] = bj;
    bcol[2 * j + 1] = log(bj);
  }
  for (int i = threadIdx.x; i < nrows; i += blockDim.x) {
    const double a = p.alpha[b * m + r0 + i];
    rstat[4 * i + 2] = a;
    rstat[4 * i + 3] = log(a);
  }
  if (nrows > 0) mbar_wait(bar, 0);
  // the integer shifts a_ij = round(G_ij log2e/eps) replace G in place; the precomputed mode's G-shifted
  // S_ij is rescaled to the same convention, S'_ij = S_ij 2^{a_ij - G_ij log2e/eps}
  for (int idx = threadIdx.x; idx < nrows * m; idx += blockDim.x) {
    const float g = Gs[idx];
    const int a = __float2int_rn(g * c2);
    if (p.pre) Cs[idx] *= ex2(fmaf(-g, c2, (float)a));   // n == 1: Cs row i holds S_i.
    As[idx] = a;
  }
  __syncthreads();

  const int cols_per_cta = (m + ncl - 1) / ncl;
  const int c0 = crank * cols_per_cta, c1 = min(m, c0 + cols_per_cta);
  const int nrw = (nrows + nwarps - 1) / nwarps;            // rows per warp (1 for C5)
  constexpr int MAXR = 2;
  // k-sums of the warp's rows for the next epilogue, accumulated in two halves of the k range so that each
  // half can cover one cluster-barrier latency
  float sacc[MAXR][VPL][4], gcr[MAXR][VPL][4];
  auto ksum_range = [&](int k_lo, int k_hi) {
    for (int rr = 0; rr < nrw && rr < MAXR; ++rr) {
      const int i = warp + rr * nwarps;
      if (i >= nrows) break;
      const float4* crow = reinterpret_cast<const float4*>(Cs + (size_t)i * n * m);
      if (p.pre) {   // NEXT-1: the row holds S_ij (n = 1); the k range is empty or [0, 1)
        if (k_lo < k_hi)
#pragma unroll
          for (int q = 0; q < VPL; ++q) {
            const int jv = q * 32 + lane;
            if (jv < mv) {
              const float4 c = crow[jv];
              sacc[rr][q][0] = c.x;
              sacc[rr][q][1] = c.y;
              sacc[rr][q][2] = c.z;
              sacc[rr][q][3] = c.w;
            }
          }
        continue;
      }
      int k = k_lo;
      // blocks of 4 k: the 16 (x VPL) MUFU.EX2 of a block are independent and issued back to back, then
      // summed in a fixed pairwise order (in-order issue would otherwise stall on each MUFU result)
      for (; k + 4 <= k_hi; k += 4) {
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
          const int jv = q * 32 + lane;
          if (jv < mv) {
            float e[4][4];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const float4 c = crow[(size_t)(k + kk) * mv + jv];
              e[kk][0] = ex2(fmaf(-c.x, c2, gcr[rr][q][0]));
              e[kk][1] = ex2(fmaf(-c.y, c2, gcr[rr][q][1]));
              e[kk][2] = ex2(fmaf(-c.z, c2, gcr[rr][q][2]));
              e[kk][3] = ex2(fmaf(-c.w, c2, gcr[rr][q][3]));
            }
#pragma unroll
            for (int v = 0; v < 4; ++v) sacc[rr][q][v] += (e[0][v] + e[1][v]) + (e[2][v] + e[3][v]);
          }
        }
      }
      for (; k < k_hi; ++k)
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
          const int jv = q * 32 + lane;
          if (jv < mv) {
            const float4 c = crow[(size_t)k * mv + jv];
            sacc[rr][q][0] += ex2(fmaf(-c.x, c2, gcr[rr][q][0]));
            sacc[rr][q][1] += ex2(fmaf(-c.y, c2, gcr[rr][q][1]));
            sacc[rr][q][2] += ex2(fmaf(-c.z, c2, gcr[rr][q][2]));
            sacc[rr][q][3] += ex2(fmaf(-c.w, c2, gcr[rr][q][3]));
          }
        }
    }
  };
  for (int rr = 0; rr < MAXR; ++rr) {
    const int i = warp + rr * nwarps;
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
      const int jv = q * 32 + lane;
      const int4 av = (i < nrows && jv < mv) ? reinterpret_cast<const int4*>(As + (size_t)i * m)[jv]
                                             : make_int4(0, 0, 0, 0);
      gcr[rr][q][0] = (float)av.x;
      gcr[rr][q][1] = (float)av.y;
      gcr[rr][q][2] = (float)av.z;
      gcr[rr][q][3] = (float)av.w;
    }
  }
  auto zero_s = [&]() {
#pragma unroll
    for (int rr = 0; rr < MAXR; ++rr)
#pragma unroll
      for (int q = 0; q < VPL; ++q)
#pragma unroll
        for (int v = 0; v < 4; ++v) sacc[rr][q][v] = 0.f;
  };
  const int khalf = n / 2;
  zero_s();
  ksum_range(0, n);                                         // k-sums of iteration 0
  int t = 0;
  bool stop = false;
  long long tr[6] = {0, 0, 0, 0, 0, 0};
  for (; t < p.iters && !stop; ++t) {
    const long long c0t = p.trace ? clock64() : 0;
    // ================= epilogues of iteration t (z_hat of iteration t-1 is complete in the replica)
    double P[VPL][4];
#pragma unroll
    for (int q = 0; q < VPL; ++q)
#pragma unroll
      for (int v = 0; v < 4; ++v) P[q][v] = 0.0;
    for (int rr = 0; rr < nrw && rr < MAXR; ++rr) {
      const int i = warp + rr * nwarps;
      if (i >= nrows) break;
      int ex[VPL][4];
      int emax = -0x7fffffff;
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const int jv = q * 32 + lane;
        const int jc = jv < mv ? jv : 0;
        const int4 a4 = reinterpret_cast<const int4*>(As + (size_t)i * m)[jc];
        const int4 k4 = reinterpret_cast<const int4*>(zk)[jc];
        ex[q][0] = k4.x - a4.x;
        ex[q][1] = k4.y - a4.y;
        ex[q][2] = k4.z - a4.z;
        ex[q][3] = k4.w - a4.w;
        if (jv < mv) emax = max(emax, max(max(ex[q][0], ex[q][1]), max(ex[q][2], ex[q][3])));
      }
      const int kM = __reduce_max_sync(0xffffffffu, emax);   // every term <= 1.42 s'_ij, the largest >= 1/2
      double tt[VPL][4];
      double lsum = 0.0;
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const int jv = q * 32 + lane;
        const int jc = jv < mv ? jv : 0;
        const double2* f2 = reinterpret_cast<const double2*>(zf) + 2 * jc;
        const double2 fa = f2[0], fb = f2[1];
        const double fz[4] = {fa.x, fa.y, fb.x, fb.y};
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          tt[q][v] = jv < mv ? ldexp_pos(sacc[rr][q][v], ex[q][v] - kM) * fz[v] : 0.0;
          lsum += tt[q][v];
        }
      }
      const double r = warp_sum(lsum);
      const double a = rstat[4 * i + 2];
      if (lane == 0) {   // w_hat_i = log alpha_i - kM_i ln2 - log r_i is formed once, after the last iteration
        rstat[4 * i + 0] = (double)kM * COT_LN2;
        rstat[4 * i + 1] = r;
      }
      const double rinv = rcp_nomufu(r);   // alpha_i / r_i
      const double rho = a * rinv;
#pragma unroll
      for (int q = 0; q < VPL; ++q)
#pragma unroll
        for (int v = 0; v < 4; ++v) P[q][v] = fma(rho, tt[q][v], P[q][v]);
    }
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
      const int jv = q * 32 + lane;
      if (jv < mv)
#pragma unroll
        for (int v = 0; v < 4; ++v) wpart[(size_t)warp * m + 4 * jv + v] = P[q][v];
    }
    const long long c1t = p.trace ? clock64() : 0;
    __syncthreads();
    for (int j = threadIdx.x; j < m; j += blockDim.x) {   // CTA partial: warps in a fixed pairwise tree
      double v16[16];
#pragma unroll
      for (int w = 0; w < 16; ++w) v16[w] = w < nwarps ? wpart[(size_t)w * m + j] : 0.0;
#pragma unroll
      for (int h = 8; h >= 1; h >>= 1)
#pragma unroll
        for (int w = 0; w < h; ++w) v16[w] += v16[w + h];
      cpart[j] = v16[0];
    }
    // ================= B1: publish the CTA partial; stream the first half of the next k-sums meanwhile
    const long long c2t = p.trace ? clock64() : 0;
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    const bool more = t + 1 < p.iters;
    zero_s();
    if (more) ksum_range(0, khalf);
    const long long c3t = p.trace ? clock64() : 0;
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    const long long c4t = p.trace ? clock64() : 0;
    // ================= column pass of this CTA's slice: one thread per (column, source CTA) in groups of 8 or
    //                   16 lanes, the ncl values combined by a fixed xor tree (deterministic), q-update written
    //                   to every replica
    const bool need = (p.tol > 0.0 && (st.iters + 1) % p.check_every == 0) || t == p.iters - 1;
    double dev = 0.0;
    const int gs_log = p.gs_log;
    for (int base = 0; base < ((c1 - c0) << gs_log); base += blockDim.x) {
      const int idx = base + threadIdx.x;
      const int jc = idx >> gs_log, src = idx & ((1 << gs_log) - 1);
      const int j = c0 + jc;
      const bool ok = jc < (c1 - c0) && src < ncl;
      double v = ok ? cluster.map_shared_rank(cpart, src)[j] : 0.0;
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      if (gs_log == 4) v += __shfl_xor_sync(0xffffffffu, v, 8);
      double zn = 0.0;
      if (ok) {
        const double bj = bcol[2 * j];
        if (src == 0) {
          dev += fabs(v - bj);
          if (!(v >= 1e-28)) s_flags = 1;
        }
        zn = zs[j] + (bcol[2 * j + 1] - log_nomufu(v));
        int kz;
        const double fz = split_z(zn, kz);
        cluster.map_shared_rank(zs, src)[j] = zn;   // lane `src` of the group writes replica `src`
        cluster.map_shared_rank(zf, src)[j] = fz;
        cluster.map_shared_rank(zk, src)[j] = kz;
      }
    }
    if (need) {
      dev = warp_sum(dev);
      __shared__ double wdev[32];
      if (lane == 0) wdev[warp] = dev;
      __syncthreads();
      if (threadIdx.x == 0) {
        double d = 0.0;
        for (int w = 0; w < nwarps; ++w) d += wdev[w];
        cluster.map_shared_rank(mon, 0)[crank] = d;
      }
    }
    // ================= B2: the q-update is in every replica; stream the second half meanwhile
    const long long c5t = p.trace ? clock64() : 0;
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    if (more) ksum_range(khalf, n);
    const long long c6t = p.trace ? clock64() : 0;
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (p.trace) {
      const long long c7t = clock64();
      tr[0] += c1t - c0t;   // epilogues
      tr[1] += c2t - c1t;   // CTA partial
      tr[2] += c3t - c2t;   // first k-sum half
      tr[3] += c4t - c3t;   // B1 wait
      tr[4] += (c5t - c4t) + (c7t - c6t);   // column pass + B2 wait
      tr[5] += c6t - c5t;   // second k-sum half
    }
    st.iters += 1;
    if (need) {
      double rr = 0.0;
      const double* m0 = cluster.map_shared_rank(mon, 0);
      for (int cr = 0; cr < ncl; ++cr) rr += m0[cr];
      st.residual = rr * (double)n;
    }
    if (p.tol > 0.0 && st.iters % p.check_every == 0 && st.residual <= p.tol) {
      st.active = 0;
      st.converged = 1;
      stop = true;
    }
  }
  // ---- write back: w_hat of this CTA's rows (from the last epilogue), z_hat (CTA 0; replicas identical)
  for (int i = threadIdx.x; i < nrows; i += blockDim.x)
    if (t > 0) p.w_hat[b * m + r0 + i] = rstat[4 * i + 3] - rstat[4 * i + 0] - log(rstat[4 * i + 1]);
  if (crank == 0) {
    for (int j = threadIdx.x; j < m; j += blockDim.x) p.z_hat[b * m + j] = zs[j];
  }
  __syncthreads();
  if (s_flags) atomicOr(&p.state[b].flags, (int)STATE_UNDERFLOW);
  if (crank == 0 && threadIdx.x == 0) {
    SolverState out = p.state[b];
    out.iters = st.iters;
    out.residual = st.residual;
    out.active = st.active;
    out.converged = st.converged;
    p.state[b] = out;
  }
  if (p.trace && threadIdx.x == 0 && b < 256)
    for (int k = 0; k < 6; ++k) p.trace[(size_t)blockIdx.x * 8 + k] = tr[k];
  cluster.sync();   // no CTA leaves while others may still read its shared memory
}

// Warp-specialised variant (m <= 128: one float4 of columns per lane; up to 2 rows per warp). The k-sums are
// iterate-independent, so NE "K" warps compute iteration t+1's s'_ij (rows w and w + NE) while NE "E" warps
// run iteration t's chain (epilogues, CTA partial, cluster barrier, column pass, cluster barrier): the MUFU work
// overlaps the latency-bound chain instead of following it. Hand-off through a shared-memory row buffer,
// written by the K warps only after the first cluster barrier of iteration t (every E warp has finished its
// epilogue of iteration t by then, so one buffer suffices), and named barrier 1 (K arrive, E sync); the E
// warps' block-level steps use named barrier 2. NE = ceil(rows / 2) (8 for the 8-CTA shape, 11 for the
// 6-CTA shape of C5). The arithmetic and every sum order are those of k_batch_cluster.
template <int NT>
__global__ void __launch_bounds__(NT, 1) k_batch_cluster_ws(BatchParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const int ncl = p.ncl;
  const int64_t b = blockIdx.x / ncl;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = p.n, m = p.m, RB = p.RB, mv = m >> 2;
  const int r0 = crank * RB;
  const int nrows = max(0, min(RB, m - r0));
  const int NE = p.ne, NET = NE * 32;                       // E warps; the other warps of the block: K warps
  const int NK = (int)(blockDim.x >> 5) - NE;
  float* Cs = reinterpret_cast<float*>(smem);
  float* Gs = Cs + (size_t)RB * n * m;
  int* As = reinterpret_cast<int*>(Gs);
  double* zs = reinterpret_cast<double*>(Gs + (size_t)RB * m);
  double* zf = zs + m;
  int* zk = reinterpret_cast<int*>(zf + m);
  double* wpart = reinterpret_cast<double*>(zk + m);
  double* cpart = wpart + (size_t)NE * m;
  double* mon = cpart + m;
  double* rstat = mon + kMaxNCL;
  double* bcol = rstat + (size_t)RB * 4;
  float* sbuf = reinterpret_cast<float*>(bcol + (size_t)m * 2);      // [RB][m] s'_ij of the next epilogue
  uint64_t* bar = reinterpret_cast<uint64_t*>(sbuf + (size_t)RB * m);
  __shared__ int s_flags;
  __shared__ double wdev[16];

  SolverState st = p.state[b];
  if (!st.active) return;
  const double inv_eps = 1.0 / p.eps[b];
  const float c2 = (float)(COT_LOG2E * inv_eps);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    s_flags = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0 && nrows > 0) {
    const uint32_t row_bytes = (uint32_t)m * 4u;
    mbar_arrive_expect_tx(bar, (uint32_t)nrows * (uint32_t)(n + 1) * row_bytes);
    const uint64_t pol = policy_evict_first();
    for (int i = 0; i < nrows; ++i) {
      for (int k = 0; k < n; ++k)
        bulk_g2s(Cs + ((size_t)i * n + k) * m, p.C + (((size_t)b * n + k) * m + r0 + i) * m, row_bytes, bar, pol);
      bulk_g2s(Gs + (size_t)i * m, p.G + ((size_t)b * m + r0 + i) * m, row_bytes, bar, pol);
    }
  }
  for (int j = threadIdx.x; j < m; j += blockDim.x) {
    zs[j] = p.z_hat[b * m + j];
    zf[j] = split_z(zs[j], zk[j]);
    const double bj = p.beta[b * m + j];
    bcol[2 * j] = bj;
    bcol[2 * j + 1] = log(bj);
  }
  for (int i = threadIdx.x; i < nrows; i += blockDim.x) {
    const double a = p.alpha[b * m + r0 + i];
    rstat[4 * i + 2] = a;
    rstat[4 * i + 3] = log(a);
  }
  if (nrows > 0) mbar_wait(bar, 0);
  for (int idx = threadIdx.x; idx < nrows * m; idx += blockDim.x) {
    const float g = Gs[idx];
    const int a = __float2int_rn(g * c2);
    if (p.pre) Cs[idx] *= ex2(fmaf(-g, c2, (float)a));
    As[idx] = a;
  }
  __syncthreads();

  const int cols_per_cta = (m + ncl - 1) / ncl;
  const int c0 = crank * cols_per_cta, c1 = min(m, c0 + cols_per_cta);
  const int kmid = n / 2;
  long long tr[6] = {0, 0, 0, 0, 0, 0};
  int t = 0;
  bool stop = false;
  // the monitor of iteration t and the freeze rule, identical in every thread (read after the second barrier)
  auto monitor = [&](bool need) {
    st.iters += 1;
    if (need) {
      double rr = 0.0;
      const double* m0 = cluster.map_shared_rank(mon, 0);
      for (int cr = 0; cr < ncl; ++cr) rr += m0[cr];
      st.residual = rr * (double)n;
    }
    if (p.tol > 0.0 && st.iters % p.check_every == 0 && st.residual <= p.tol) {
      st.active = 0;
      st.converged = 1;
      stop = true;
    }
  };
  if (warp >= NE) {
    // ============================================================== K warps: s'_ij of the next iteration
    const int w = warp - NE;   // rows w, w + NK, w + 2 NK, w + 3 NK
    float gcr[4][4], s[4][4];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const int i = w + rr * NK;
      const int4 av = (i < nrows && lane < mv) ? reinterpret_cast<const int4*>(As + (size_t)i * m)[lane]
                                               : make_int4(0, 0, 0, 0);
      gcr[rr][0] = (float)av.x;
      gcr[rr][1] = (float)av.y;
      gcr[rr][2] = (float)av.z;
      gcr[rr][3] = (float)av.w;
    }
    auto zero = [&]() {
#pragma unroll
      for (int rr = 0; rr < 4; ++rr)
#pragma unroll
        for (int v = 0; v < 4; ++v) s[rr][v] = 0.f;
    };
    auto ksum = [&](int k_lo, int k_hi) {
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        const int i = w + rr * NK;
        if (i >= nrows || lane >= mv) continue;
        const float4* crow = reinterpret_cast<const float4*>(Cs + (size_t)i * n * m);
        if (p.pre) {
          if (k_lo < k_hi) {
            const float4 c = crow[lane];
            s[rr][0] = c.x;
            s[rr][1] = c.y;
            s[rr][2] = c.z;
            s[rr][3] = c.w;
          }
          continue;
        }
        int k = k_lo;
        for (; k + 4 <= k_hi; k += 4) {
          float e[4][4];
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const float4 c = crow[(size_t)(k + kk) * mv + lane];
            e[kk][0] = ex2(fmaf(-c.x, c2, gcr[rr][0]));
            e[kk][1] = ex2(fmaf(-c.y, c2, gcr[rr][1]));
            e[kk][2] = ex2(fmaf(-c.z, c2, gcr[rr][2]));
            e[kk][3] = ex2(fmaf(-c.w, c2, gcr[rr][3]));
          }
#pragma unroll
          for (int v = 0; v < 4; ++v) s[rr][v] += (e[0][v] + e[1][v]) + (e[2][v] + e[3][v]);
        }
        for (; k < k_hi; ++k) {
          const float4 c = crow[(size_t)k * mv + lane];
          s[rr][0] += ex2(fmaf(-c.x, c2, gcr[rr][0]));
          s[rr][1] += ex2(fmaf(-c.y, c2, gcr[rr][1]));
          s[rr][2] += ex2(fmaf(-c.z, c2, gcr[rr][2]));
          s[rr][3] += ex2(fmaf(-c.w, c2, gcr[rr][3]));
        }
      }
    };
    auto publish = [&]() {   // s' rows into sbuf, then named barrier 1 (arrive: no wait)
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        const int i = w + rr * NK;
        if (i < nrows && lane < mv)
          reinterpret_cast<float4*>(sbuf + (size_t)i * m)[lane] = make_float4(s[rr][0], s[rr][1], s[rr][2], s[rr][3]);
      }
      __threadfence_block();
      asm volatile("bar.arrive 1, %0;" ::"r"(blockDim.x) : "memory");
    };
    zero();
    ksum(0, n);
    publish();
    for (; t < p.iters && !stop; ++t) {
      const bool more = t + 1 < p.iters;
      const bool need = (p.tol > 0.0 && (st.iters + 1) % p.check_every == 0) || t == p.iters - 1;
      const long long k0 = p.trace ? clock64() : 0;
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      zero();
      if (more) ksum(0, kmid);
      const long long k1 = p.trace ? clock64() : 0;
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      const long long k2 = p.trace ? clock64() : 0;
      if (more) ksum(kmid, n);
      const long long k3 = p.trace ? clock64() : 0;
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
      monitor(need);
      if (more && !stop) publish();   // after B1 of iteration t: the E warps are done with sbuf
      if (p.trace) {
        tr[2] += k1 - k0;
        tr[5] += k3 - k2;
      }
    }
  } else {
    // ============================================================== E warps: the iteration chain
    const int et = threadIdx.x;
    for (; t < p.iters && !stop; ++t) {
      const bool need = (p.tol > 0.0 && (st.iters + 1) % p.check_every == 0) || t == p.iters - 1;
      asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x) : "memory");   // s'(t) is in sbuf
      const long long c0t = p.trace ? clock64() : 0;
      const float* sb = sbuf;
      // the warp's two rows side by side (independent shuffle / reduction chains overlap)
      double P[4] = {0.0, 0.0, 0.0, 0.0};
      {
        const int jc = lane < mv ? lane : 0;
        const int4 k4 = reinterpret_cast<const int4*>(zk)[jc];
        const double2* f2 = reinterpret_cast<const double2*>(zf) + 2 * jc;
        const double2 fa = f2[0], fb = f2[1];
        const double fz[4] = {fa.x, fa.y, fb.x, fb.y};
        bool valid[2];
        int ex[2][4], kM[2];
        double tt[2][4], lsum[2];
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int i = warp + rr * NE;
          valid[rr] = i < nrows;
          const int ic = valid[rr] ? i : 0;
          const int4 a4 = reinterpret_cast<const int4*>(As + (size_t)ic * m)[jc];
          ex[rr][0] = k4.x - a4.x;
          ex[rr][1] = k4.y - a4.y;
          ex[rr][2] = k4.z - a4.z;
          ex[rr][3] = k4.w - a4.w;
          const int emax = lane < mv ? max(max(ex[rr][0], ex[rr][1]), max(ex[rr][2], ex[rr][3])) : -0x7fffffff;
          kM[rr] = __reduce_max_sync(0xffffffffu, emax);
          const float4 s4 = reinterpret_cast<const float4*>(sb + (size_t)ic * m)[jc];
          const float sv[4] = {s4.x, s4.y, s4.z, s4.w};
          lsum[rr] = 0.0;
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            tt[rr][v] = lane < mv && valid[rr] ? ldexp_pos(sv[v], ex[rr][v] - kM[rr]) * fz[v] : 0.0;
            lsum[rr] += tt[rr][v];
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          lsum[0] += __shfl_xor_sync(0xffffffffu, lsum[0], o);
          lsum[1] += __shfl_xor_sync(0xffffffffu, lsum[1], o);
        }
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          if (!valid[rr]) continue;
          const int i = warp + rr * NE;
          const double r = lsum[rr];
          if (lane == 0) {
            rstat[4 * i + 0] = (double)kM[rr] * COT_LN2;
            rstat[4 * i + 1] = r;
          }
          const double rho = rstat[4 * i + 2] * rcp_nomufu(r);
#pragma unroll
          for (int v = 0; v < 4; ++v) P[v] = fma(rho, tt[rr][v], P[v]);
        }
      }
      if (lane < mv)
#pragma unroll
        for (int v = 0; v < 4; ++v) wpart[(size_t)warp * m + 4 * lane + v] = P[v];
      const long long c1t = p.trace ? clock64() : 0;
      asm volatile("bar.sync 2, %0;" ::"r"(NET) : "memory");
      for (int j = et; j < m; j += NET) {   // CTA partial: the E warps in a fixed pairwise tree
        double v16[16];
#pragma unroll
        for (int w = 0; w < 16; ++w) v16[w] = w < NE ? wpart[(size_t)w * m + j] : 0.0;
#pragma unroll
        for (int h = 8; h >= 1; h >>= 1)
#pragma unroll
          for (int w = 0; w < h; ++w) v16[w] += v16[w + h];
        cpart[j] = v16[0];
      }
      const long long c2t = p.trace ? clock64() : 0;
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
      const long long c4t = p.trace ? clock64() : 0;
      double dev = 0.0;
      for (int base = 0; base < ((c1 - c0) << 3); base += NET) {
        const int idx = base + et;
        const int jc = idx >> 3, src = idx & 7;
        const int j = c0 + jc;
        const bool ok = jc < (c1 - c0) && src < ncl;
        double v = ok ? cluster.map_shared_rank(cpart, src)[j] : 0.0;
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        if (ok) {
          const double bj = bcol[2 * j];
          if (src == 0) {
            dev += fabs(v - bj);
            if (!(v >= 1e-28)) s_flags = 1;
          }
          const double zn = zs[j] + (bcol[2 * j + 1] - log_nomufu(v));
          int kz;
          const double fzn = split_z(zn, kz);
          cluster.map_shared_rank(zs, src)[j] = zn;
          cluster.map_shared_rank(zf, src)[j] = fzn;
          cluster.map_shared_rank(zk, src)[j] = kz;
        }
      }
      if (need) {
        dev = warp_sum(dev);
        if (lane == 0) wdev[warp] = dev;
        asm volatile("bar.sync 2, %0;" ::"r"(NET) : "memory");
        if (et == 0) {
          double d = 0.0;
          for (int w = 0; w < NE; ++w) d += wdev[w];
          cluster.map_shared_rank(mon, 0)[crank] = d;
        }
      }
      const long long c5t = p.trace ? clock64() : 0;
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
      monitor(need);
      if (p.trace) {
        const long long c7t = clock64();
        tr[0] += c1t - c0t;
        tr[1] += c2t - c1t;
        tr[3] += c4t - c2t;
        tr[4] += c7t - c5t + (c5t - c4t);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nrows; i += blockDim.x)
    if (t > 0) p.w_hat[b * m + r0 + i] = rstat[4 * i + 3] - rstat[4 * i + 0] - log(rstat[4 * i + 1]);
  if (crank == 0)
    for (int j = threadIdx.x; j < m; j += blockDim.x) p.z_hat[b * m + j] = zs[j];
  __syncthreads();
  if (s_flags) atomicOr(&p.state[b].flags, (int)STATE_UNDERFLOW);
  if (crank == 0 && threadIdx.x == 0) {
    SolverState out = p.state[b];
    out.iters = st.iters;
    out.residual = st.residual;
    out.active = st.active;
    out.converged = st.converged;
    p.state[b] = out;
  }
  if (p.trace && b < 256) {
    unsigned long long* tp = p.trace + (size_t)blockIdx.x * 8;
    if (threadIdx.x == 0) {
      tp[0] = tr[0];
      tp[1] = tr[1];
      tp[3] = tr[3];
      tp[4] = tr[4];
    }
    if (threadIdx.x == NET) {
      tp[2] = tr[2];
      tp[5] = tr[5];
    }
  }
  cluster.sync();
}

static size_t batch_smem_bytes(int n, int m, int RB, int nwarps) {
  return (size_t)RB * n * m * 4 + (size_t)RB * m * 4 + (size_t)m * 20 + (size_t)nwarps * m * 8 + (size_t)m * 8 +
         kMaxNCL * 8 + (size_t)RB * 32 + (size_t)m * 16 + 16;
}

// Cluster shapes. Measured on B200 (scripts/ubench/clocc.cu, ubench_batch.py, ubench_c2.py): with one CTA of
// ~200 KB per SM only 15 clusters of 8 CTAs are co-resident (GPC packing: 120 of 148 SMs), but 22 clusters of 6;
// C5 (4096 problems) runs 12% faster as 6-CTA clusters of 11 warps (2 rows per warp, balanced k-sums) than as
// 8-CTA clusters, while a batch that fits in one wave of 8-CTA clusters (C2) is latency-bound and keeps the
// 8-CTA shape (fewer rows per CTA). A shape is feasible when a CTA's rows fit (<= 2 rows per warp) and its
// shared memory fits the per-SM budget of its occupancy.
struct ClusterShape {
  int ncl, threads, ctas_per_sm;
};
constexpr ClusterShape kShapes[] = {{8, 512, 1}, {6, 352, 1}, {12, 256, 2}, {16, 256, 2}, {6, 512, 1}};
constexpr int kLatencyShape = 0, kThroughputShape = 1;

struct BatchCfg {
  ClusterShape sh;
  int RB, threads, ne;
  bool ws;   // warp-specialised kernel (threads = 2 x 32 x ceil(rows / 2))
  size_t smem;
  void* fn;
};

static bool shape_config(int k, int64_t n, int64_t m, BatchCfg* out) {
  const ClusterShape sh = kShapes[k];
  if (m < sh.ncl) return false;
  const int RB = (int)((m + sh.ncl - 1) / sh.ncl);
  const int nwarps = sh.threads / 32;
  if (RB > 2 * nwarps) return false;
  const size_t smem = batch_smem_bytes((int)n, (int)m, RB, std::min(RB, nwarps));
  const size_t budget = sh.ctas_per_sm == 1 ? 226 * 1024 : 110 * 1024;   // of 227 KB per CTA, 228 KB per SM
  if (smem > budget) return false;
  out->sh = sh;
  out->RB = RB;
  out->smem = smem;
  // 1 CTA per SM and m <= 128 (<= 22 rows per CTA): warp-specialised, NE = ceil(rows / 2) epilogue warps and as
  // many k-sum warps (COT_BATCH_WS=0: the interleaved kernel)
  const char* wsv = getenv("COT_BATCH_WS");
  out->ws = sh.ctas_per_sm == 1 && m <= 128 && RB <= 22 && !(wsv && atoi(wsv) == 0);
  if (out->ws) {
    const int ne = (RB + 1) / 2;
    int kr = 2;   // rows per k-sum warp (COT_BATCH_KR: 1..4; 2 measured best on C5 and C2)
    if (const char* ev = getenv("COT_BATCH_KR")) kr = std::max(1, std::min(4, atoi(ev)));
    const int nk = (RB + kr - 1) / kr;
    out->ne = ne;
    out->threads = 32 * (ne + nk);
    out->smem = batch_smem_bytes((int)n, (int)m, RB, ne) + (size_t)RB * m * 4;
    if (out->smem > budget) return false;
    out->fn = out->threads <= 512 ? (void*)k_batch_cluster_ws<512>
                                  : out->threads <= 576 ? (void*)k_batch_cluster_ws<576> : (void*)k_batch_cluster_ws<704>;
    return true;
  }
  out->threads = std::min(RB, nwarps) * 32;
  const bool v1 = m <= 128;
  if (sh.ctas_per_sm == 1)
    out->fn = v1 ? (void*)k_batch_cluster<1, 512, 1> : (void*)k_batch_cluster<2, 512, 1>;
  else
    out->fn = v1 ? (void*)k_batch_cluster<1, 256, 2> : (void*)k_batch_cluster<2, 256, 2>;
  return true;
}

// co-resident clusters of a configuration (cached per shared-memory size)
static int active_clusters(const BatchCfg& c) {
  static std::mutex mu;   // calls on distinct streams may run concurrently (include/cyclicot.h)
  static int64_t cached_key = -1;
  static int cached = 0;
  const int64_t key = ((int64_t)c.smem * 64 + c.sh.ncl) * 2 + (c.ws ? 1 : 0);
  std::lock_guard<std::mutex> lock(mu);
  if (key == cached_key) return cached;
  cudaFuncSetAttribute(c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem);
  if (c.sh.ncl > 8) cudaFuncSetAttribute(c.fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(c.sh.ncl * 64));
  cfg.blockDim = dim3((unsigned)c.threads);
  cfg.dynamicSmemBytes = c.smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = c.sh.ncl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, c.fn, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  cached_key = key;
  cached = n;
  return n;
}

// The shape for a batch of B problems: the latency shape while the batch fits in one wave of it, else the
// throughput shape; then any feasible shape. COT_BATCH_SHAPE forces one (experiments).
static bool batch_config(int64_t n, int64_t m, int64_t B, BatchCfg* out) {
  if (const char* ev = getenv("COT_BATCH_SHAPE")) {
    const int k = atoi(ev);
    return k >= 0 && k < (int)(sizeof(kShapes) / sizeof(kShapes[0])) && shape_config(k, n, m, out);
  }
  BatchCfg lat;
  const bool have_lat = shape_config(kLatencyShape, n, m, &lat);
  if (have_lat && (B <= 0 || B <= active_clusters(lat))) {
    *out = lat;
    return true;
  }
  if (shape_config(kThroughputShape, n, m, out)) return true;
  if (have_lat) {
    *out = lat;
    return true;
  }
  for (int k = 0; k < (int)(sizeof(kShapes) / sizeof(kShapes[0])); ++k)
    if (shape_config(k, n, m, out)) return true;
  return false;
}

bool batch_cluster_eligible(const IterArgs& a) {
  if (batch_chain_eligible(a)) return true;
  if (a.dtype != COT_F32 || a.m % 4 != 0 || a.m > 256 || a.R != a.m || (a.flags & (COT_FORCE_LDG | COT_FORCE_TMA)))
    return false;
  BatchCfg c;
  return batch_config(a.n, a.m, 0, &c);
}

cudaError_t launch_batch_cluster(const IterArgs& a, const Workspace& ws, int iters, cudaStream_t s) {
  if (batch_chain_eligible(a)) return launch_batch_chain(a, ws, iters, s);
  BatchCfg bc;
  if (!batch_config(a.n, a.m, a.B, &bc)) return cudaErrorInvalidConfiguration;
  BatchParams p;
  p.C = static_cast<const float*>(a.C);
  p.G = static_cast<const float*>(a.G);
  p.alpha = a.alpha;
  p.beta = a.beta;
  p.w_hat = a.w_hat;
  p.z_hat = a.z_hat;
  p.eps = a.eps;
  p.state = ws.state;
  p.n = (int)a.n;
  p.m = (int)a.m;
  p.RB = bc.RB;
  p.ncl = bc.sh.ncl;
  p.gs_log = bc.sh.ncl <= 8 ? 3 : 4;
  p.ne = bc.ws ? bc.ne : 0;
  p.iters = iters;
  p.tol = a.tol;
  p.check_every = a.check_every > 0 ? a.check_every : 1;
  p.pre = (a.flags & COT_PRECOMPUTED) ? 1 : 0;
  void* fn = bc.fn;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bc.smem);
  if (e != cudaSuccess) return e;
  if (p.ncl > 8) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.B * p.ncl));
  cfg.blockDim = dim3((unsigned)bc.threads);
  cfg.dynamicSmemBytes = bc.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.ncl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static unsigned long long* trace_buf = nullptr;   // diagnostics only (COT_TRACE=1)
  p.trace = nullptr;
  if (getenv("COT_TRACE")) {
    if (!trace_buf) cudaMalloc(&trace_buf, 256 * kMaxNCL * 8 * sizeof(unsigned long long));
    cudaMemsetAsync(trace_buf, 0, 256 * kMaxNCL * 8 * sizeof(unsigned long long), s);
    p.trace = trace_buf;
  }
  void* args[] = {&p};
  e = cudaLaunchKernelExC(&cfg, fn, args);
  if (e == cudaSuccess && p.trace) {
    const int ctas = (int)std::min<int64_t>(a.B, 256) * p.ncl;
    std::vector<unsigned long long> h((size_t)ctas * 8);
    cudaStreamSynchronize(s);
    cudaMemcpy(h.data(), p.trace, h.size() * 8, cudaMemcpyDeviceToHost);
    double acc[6] = {0};
    for (int c = 0; c < ctas; ++c)
      for (int k = 0; k < 6; ++k) acc[k] += (double)h[(size_t)c * 8 + k] / ctas / std::max(iters, 1);
    int act = -1;
    cudaOccupancyMaxActiveClusters(&act, fn, &cfg);
    fprintf(stderr, "[cot batch trace] cluster %d x %d threads, %d co-resident clusters; per-iter cycles: epilogue "
            "%.0f cta_partial %.0f ksum1 %.0f B1_wait %.0f colpass+B2_wait %.0f ksum2 %.0f\n", p.ncl,
            (int)cfg.blockDim.x, act, acc[0], acc[1], acc[2], acc[3], acc[4], acc[5]);
  }
  return e;
}

}  // namespace cot
