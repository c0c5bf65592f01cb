// K-ITER (TMA path): a persistent, warp-specialised cyclic Sinkhorn kernel for one problem (B == 1) with
// fp32 costs and m % 4 == 0. Same arithmetic as k_rows_ldg + k_cols (k_iter.cu), organised for HBM.
// Three warp roles per CTA (one CTA per SM, one unit of consecutive rows per CTA):
//
//   producer warp (1 elected lane): streams the CTA's rows of C through an NSLOT-deep ring of shared-
//     memory slots with 1-D TMA bulk copies (cp.async.bulk, SASS UBLKCP); a slot holds KS consecutive
//     k-rows C[k][i][0..m) of one row i; completion via mbarrier transaction counts (full[]), reuse via
//     consumer-warp arrivals (empty[]). It never depends on the potentials, so it runs ahead across
//     epilogues, device-wide syncs and iteration boundaries.
//   consumer warps (VEC consecutive columns per thread): per row, the streamed k-sum
//     s_ij = sum_k exp2((G_ij - C_ijk) * log2e/eps) (one FFMA + one MUFU.EX2 + one FADD per element), then
//     the fp64 epilogue: x_ij = z_hat_j - G_ij/eps, r_i = sum_j s_ij exp(x_ij - M'_i) and M_i = max_j x_ij in
//     ONE combined block reduction against the previous iteration's row maximum M'_i (exact exponent split:
//     no precision cost), w_hat_i = log alpha_i - M'_i - log r_i, P_j += (alpha_i / r_i) s_ij exp(x_ij - M'_i).
//     Rows whose potentials are not ready yet (the previous q-update is still in flight) are parked in
//     shared memory; k-sums run at most one iteration ahead of epilogues.
//   sync warp: owns every device-wide step, off the consumers' critical path: waits for the consumers to
//     publish the CTA's column partial (bar.arrive / bar.sync), arrives on device barrier B1, reduces this
//     CTA's slice of columns over all units in a fixed order (deterministic), applies the q-update
//     z_hat_j += log beta_j - log c_j, arrives on B2, evaluates the monitor / freeze rule, and publishes the
//     new z generation to the consumers through shared memory (st.release / ld.acquire at CTA scope).
//
// The grid is co-resident (cooperative launch). With rows_only = 1 the kernel performs only the row pass
// of one iteration (no device-wide steps): cerot_rows.
#include "common.cuh"
#include "internal.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace cot {

struct TmaParams {
  const float* C;        // [n][R][m]
  const float* G;        // [R][m]
  const double* alpha;   // [m]
  const double* beta;    // [m]
  double* w_hat;         // [m]
  double* z_hat;         // [m]
  const double* eps;     // [1]
  int n, m, R, row_begin, rpu, U;
  int KS, nslot;
  int iters;
  int rows_only;
  double tol;
  long long check_every;
  double* partials;      // [U][m]
  double* resid_part;    // [gridDim.x]
  SolverState* state;    // [1]
  unsigned* bar;         // [4]: two device-wide barriers {arrival count, generation}
  int nk, ne, qn;        // k-sum warps, epilogue warps, row-queue depth
  int evict_last_rows;   // rows [0, evict_last_rows) of every block are streamed with an L2 evict_last hint
  int diag;              // COT_DIAG_* bits (diagnostics only)
  int pre;               // precomputed mode (NEXT-1): C is S [R][m] (n = 1) and s_ij = S_ij
  unsigned long long* trace;   // diagnostics: [grid][8] cycle counters, or nullptr
};

__device__ __forceinline__ void cbar(int nthreads) {   // consumer-only named barrier
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned x) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(x) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_release(unsigned* p, unsigned x) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(x) : "memory");
}
__device__ __forceinline__ void st_relaxed(unsigned* p, unsigned x) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(x) : "memory");
}
__device__ __forceinline__ unsigned lds_volatile(const unsigned* p) { return *(volatile const unsigned*)p; }
__device__ __forceinline__ unsigned lds_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void sts_release(unsigned* p, unsigned v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
// Hand-off barrier between the consumer warps (arrive, non-blocking) and the sync warp (sync).
__device__ __forceinline__ void handoff_arrive(int nthreads) {
  asm volatile("bar.arrive 2, %0;" ::"r"(nthreads) : "memory");
}
__device__ __forceinline__ void handoff_sync(int nthreads) {
  asm volatile("bar.sync 2, %0;" ::"r"(nthreads) : "memory");
}

// Device-wide barrier among the consumer warps of all CTAs, split into arrive / wait so that independent
// work can run in between. bar = {arrival count, generation}. Ordering uses release/acquire atomics at gpu
// scope (the CTA barrier before the arrival makes it cumulative over the CTA's writes); no fence.sc, which
// would also stall this SM's in-flight TMA traffic.
__device__ __forceinline__ unsigned grid_arrive(unsigned* bar, int nct, unsigned* gen_sh) {
  cbar(nct);
  if (threadIdx.x == 0) {
    const unsigned gen = ld_acquire(bar + 1);
    const unsigned arrived = atom_add_acq_rel(bar, 1u);
    if (arrived == gridDim.x - 1) {
      st_relaxed(bar, 0u);
      red_add_release(bar + 1, 1u);
    }
    *gen_sh = gen;
  }
  cbar(nct);
  return *gen_sh;
}
__device__ __forceinline__ void grid_wait(unsigned* bar, unsigned gen, int nct) {
  if (threadIdx.x == 0) {
    while (ld_acquire(bar + 1) == gen) __nanosleep(20);
  }
  cbar(nct);
}

// Two-cbar block reduction for rare uses (monitor partial).
__device__ __forceinline__ double cblk_sum(double v, double* sh, int nct) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) sh[wid] = v;
  cbar(nct);
  double t = 0.0;
  for (int w = 0; w < (nct >> 5); ++w) t += sh[w];
  cbar(nct);
  return t;
}
// One-cbar block reductions for the epilogues: double-buffered scratch (`buf` alternates; the next
// reduction's cbar orders every read of this buffer before its reuse two reductions later).
__device__ __forceinline__ void cblk_maxsum(double& mx, double& sm, double* red2, int& buf, int nct,
                                            int wbase) {
  const int lane = threadIdx.x & 31, wid = (threadIdx.x >> 5) - wbase;   // warp index within the group
  mx = warp_max(mx);
  sm = warp_sum(sm);
  double* r = red2 + buf * 64;
  if (lane == 0) {
    r[wid] = mx;
    r[32 + wid] = sm;
  }
  cbar(nct);
  double M = r[0], S = r[32];
  for (int w = 1; w < (nct >> 5); ++w) {
    M = fmax(M, r[w]);
    S += r[32 + w];
  }
  mx = M;
  sm = S;
  buf ^= 1;
}
__device__ __forceinline__ double cblk_max1(double v, double* red2, int& buf, int nct, int wbase) {
  double s = 0.0;
  cblk_maxsum(v, s, red2, buf, nct, wbase);
  return v;
}
__device__ __forceinline__ double cblk_sum1(double v, double* red2, int& buf, int nct, int wbase) {
  double m = -INFINITY;
  cblk_maxsum(m, v, red2, buf, nct, wbase);
  return v;
}

// exp(d) for d in fp64, |d| < ~700: 2^(round) exactly in fp64 times MUFU 2^frac with |frac| <= 1/2, so the
// fp32 rounding of the argument costs < 3e-8 relative regardless of |d|.
__device__ __forceinline__ double exp_split(double d) {
  const double a = d * COT_LOG2E;
  const double ai = fmax(rint(a), -1022.0);   // below 2^-1022: f is very negative and ex2(f) flushes to 0
  const float f = (float)(a - ai);
  const long long e = (long long)ai + 1023;
  return (double)ex2(f) * __longlong_as_double(e << 52);
}

template <int VEC>
struct VecF;
template <>
struct VecF<2> {
  using type = float2;
  __device__ static void get(const type& v, float* o) { o[0] = v.x; o[1] = v.y; }
  __device__ static type make(const float* o) { return make_float2(o[0], o[1]); }
};
template <>
struct VecF<4> {
  using type = float4;
  __device__ static void get(const type& v, float* o) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
  __device__ static type make(const float* o) { return make_float4(o[0], o[1], o[2], o[3]); }
};

template <int CPT, int EPT, int KS>
__global__ void __launch_bounds__(448, 1) k_iter_tma(TmaParams p) {
  constexpr int VEC = 4;
  using VT = float4;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = p.nk, ne = p.ne;             // k-sum warps, epilogue warps; then producer, sync warps
  const int nkt = nk * 32, net = ne * 32;
  const int wprod = nk + ne, wsync = nk + ne + 1;
  const int m = p.m, mv = m / VEC;
  const int n = p.n, R = p.R;
  const int U = p.U, rpu = p.rpu, QN = p.qn;
  const size_t slot_floats = (size_t)KS * m;
  // ---- shared memory layout
  float* ring = reinterpret_cast<float*>(smem);
  float* queue = reinterpret_cast<float*>(smem + (size_t)p.nslot * slot_floats * 4 + 1024);   // [QN][m]
  double* rowstat = reinterpret_cast<double*>(queue + (size_t)QN * m);   // [rpu][4]: M', M, r, log alpha
  uint64_t* full = reinterpret_cast<uint64_t*>(rowstat + (size_t)rpu * 4);
  uint64_t* empty = full + p.nslot;
  uint64_t* qfull = empty + p.nslot;
  uint64_t* qempty = qfull + QN;
  unsigned* ctl = reinterpret_cast<unsigned*>(qempty + QN);
  // ctl: [0] TMA slots issued [1] producer done [2] stop producer [4] z generation (completed q-updates)
  //      [5] halt (frozen) [6] rows produced by the k-sum warps [7] k-sum warps done
  //      [8] k-sum broadcast [9] epilogue broadcast
  double* red2 = reinterpret_cast<double*>(ctl + 16);   // [2][64]

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.nslot; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nk);
    }
    for (int q = 0; q < QN; ++q) {
      mbar_init(&qfull[q], nk);
      mbar_init(&qempty[q], ne);
    }
    for (int c = 0; c < 16; ++c) ctl[c] = 0;
    fence_mbar_init();
  }
  __syncthreads();

  const int u = blockIdx.x;                 // one unit of rows per CTA (the launcher sets grid == U)
  const int i0 = u * rpu, i1 = min(R, i0 + rpu), nrows = i1 - i0;
  const bool active0 = p.state[0].active != 0;
  const double inv_eps = 1.0 / p.eps[0];

  if (warp == wprod) {
    // ===================================================================== producer (one lane)
    if (lane == 0 && active0) {
      const uint64_t pol_first = policy_evict_first();
      const uint64_t pol_last = policy_evict_last();
      uint32_t slot = 0, phase = 0;
      unsigned issued = 0;
      long long prod_wait = 0;
      const long long tp0 = clock64();
      const uint32_t row_bytes = (uint32_t)m * 4u;
      for (int t = 0; t < p.iters; ++t) {
        for (int i = i0; i < i1; ++i) {
          const uint64_t pol = i < p.evict_last_rows ? pol_last : pol_first;
          for (int k0 = 0; k0 < n; k0 += KS) {
            if (lds_volatile(&ctl[2])) goto producer_done;
            const int kk = min(KS, n - k0);
            const long long tw0 = p.trace ? clock64() : 0;
            mbar_wait(&empty[slot], phase ^ 1u);
            if (p.trace) prod_wait += clock64() - tw0;
            mbar_arrive_expect_tx(&full[slot], (uint32_t)kk * row_bytes);
            float* dst = ring + (size_t)slot * slot_floats;
            for (int q = 0; q < kk; ++q)
              bulk_g2s(dst + (size_t)q * m, p.C + ((size_t)(k0 + q) * R + i) * m, row_bytes, &full[slot], pol);
            ++issued;
            *(volatile unsigned*)&ctl[0] = issued;
            if (++slot == (uint32_t)p.nslot) {
              slot = 0;
              phase ^= 1u;
            }
          }
        }
      }
    producer_done:
      if (p.trace) {
        p.trace[blockIdx.x * 8 + 0] = prod_wait;
        p.trace[blockIdx.x * 8 + 1] = clock64() - tp0;
      }
    }
    if (lane == 0) {
      __threadfence_block();
      *(volatile unsigned*)&ctl[1] = 1u;
    }
    __syncwarp();
  } else if (warp == wsync) {
    // ===================================================================== sync warp
    // Per iteration t: wait until the epilogue warps published the CTA's column partial of t; B1; column
    // pass of this CTA's slice; B2; monitor / freeze rule; publish z generation t+1 (or halt).
    SolverState st = p.state[0];
    const long long iters0 = st.iters;
    const bool sync = !p.rows_only && !(p.diag & COT_DIAG_NO_SYNC);
    const int cols_per_cta = (m + gridDim.x - 1) / gridDim.x;
    const int col0 = blockIdx.x * cols_per_cta;
    const int col1 = min(m, col0 + cols_per_cta);
    if (!p.rows_only && active0) {
      for (int t = 0; t < p.iters; ++t) {
        handoff_sync(net + 32);               // epilogue warps published partial t (and w_hat of t)
        if (!sync) {
          st.iters += 1;
          if (lane == 0) sts_release(&ctl[4], (unsigned)(t + 1));
          continue;
        }
        // ---- B1: every CTA's partial of iteration t is published
        if (lane == 0) {
          const unsigned gen = ld_acquire(p.bar + 1);
          if (atom_add_acq_rel(p.bar, 1u) == gridDim.x - 1) {
            st_relaxed(p.bar, 0u);
            red_add_release(p.bar + 1, 1u);
          }
          while (ld_acquire(p.bar + 1) == gen) __nanosleep(20);
        }
        __syncwarp();
        // ---- column pass: c_j = sum_u P_uj (fixed order: lane-strided units, then the warp_sum tree)
        const long long itg = iters0 + t + 1;
        const bool need_resid = (p.tol > 0.0 && itg % p.check_every == 0) || t == p.iters - 1;
        double dev = 0.0;
        for (int cb = col0; cb < col1; cb += 8) {
          double acc[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[c] = 0.0;
          for (int u2 = lane; u2 < U; u2 += 32) {
#pragma unroll
            for (int c = 0; c < 8; ++c)
              if (cb + c < col1) acc[c] += __ldcg(p.partials + (size_t)u2 * m + cb + c);
          }
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[c] = warp_sum(acc[c]);
          const int c = lane;
          if (c < 8 && cb + c < col1) {
            double cj = acc[0];
#pragma unroll
            for (int q = 1; q < 8; ++q) cj = (c == q) ? acc[q] : cj;
            const int j = cb + c;
            const double bj = p.beta[j];
            dev += fabs(cj - bj);
            if (!(cj >= 1e-28)) atomicOr(&p.state[0].flags, (int)STATE_UNDERFLOW);
            p.z_hat[j] = __ldcg(p.z_hat + j) + (log(bj) - log(cj));
          }
        }
        dev = warp_sum(dev);
        // ---- B2: every q-update of iteration t is written
        if (lane == 0) {
          if (need_resid) p.resid_part[blockIdx.x] = dev;
          const unsigned gen = ld_acquire(p.bar + 3);
          if (atom_add_acq_rel(p.bar + 2, 1u) == gridDim.x - 1) {
            st_relaxed(p.bar + 2, 0u);
            red_add_release(p.bar + 3, 1u);
          }
          while (ld_acquire(p.bar + 3) == gen) __nanosleep(20);
        }
        __syncwarp();
        st.iters += 1;
        if (need_resid) {   // every CTA sums the monitor partials in the same order
          double r = 0.0;
          for (int b2 = lane; b2 < (int)gridDim.x; b2 += 32) r += __ldcg(p.resid_part + b2);
          st.residual = warp_sum(r) * (double)n;
        }
        if (p.tol > 0.0 && st.iters % p.check_every == 0 && st.residual <= p.tol) {
          st.active = 0;
          st.converged = 1;
          if (lane == 0) sts_release(&ctl[5], 1u);   // halt: iteration t+1 is discarded
          break;
        }
        if (lane == 0) sts_release(&ctl[4], (unsigned)(t + 1));
      }
      if (blockIdx.x == 0 && lane == 0) {
        SolverState out = p.state[0];
        out.iters = st.iters;
        out.residual = st.residual;
        out.active = st.active;
        out.converged = st.converged;
        p.state[0] = out;
      }
    }
  } else if (warp < nk) {
    // ===================================================================== k-sum warps
    // s_ij = sum_k exp2((G_ij - C_ijk) log2e/eps) for every row, streamed from the TMA ring into the row
    // queue; never waits for the potentials. Threads past the last column compute (in-bounds) garbage that
    // the epilogue masks out, so the slot body has no per-column branches.
    const int kt = threadIdx.x;
    const float c2 = (float)(COT_LOG2E * inv_eps);
    uint32_t slot = 0, phase = 0, qs = 0, qph = 0;
    unsigned consumed = 0, produced = 0;
    long long c_ksum = 0;
    VT gnext[CPT];
    auto load_g = [&](int row) {
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const int jv = q * nkt + kt;
        gnext[q] = jv < mv ? __ldg(reinterpret_cast<const VT*>(p.G + (size_t)row * m) + jv)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    auto release = [&]() {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      ++consumed;
      if (++slot == (uint32_t)p.nslot) {
        slot = 0;
        phase ^= 1u;
      }
    };
    if (active0) load_g(i0);
    const int total_rows = p.iters * nrows;
    for (int rr = 0; active0 && rr < total_rows; ++rr) {
      // CTA-uniform (k-sum warps) check of the halt flag
      if (kt == 0) ctl[8] = lds_acquire(&ctl[5]);
      asm volatile("bar.sync 3, %0;" ::"r"(nkt) : "memory");
      const bool halt = ctl[8] != 0;
      asm volatile("bar.sync 3, %0;" ::"r"(nkt) : "memory");
      if (halt) break;
      const int r = rr % nrows;
      float gc[CPT][VEC], s[CPT][VEC];
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        gc[q][0] = gnext[q].x * c2;
        gc[q][1] = gnext[q].y * c2;
        gc[q][2] = gnext[q].z * c2;
        gc[q][3] = gnext[q].w * c2;
#pragma unroll
        for (int v = 0; v < VEC; ++v) s[q][v] = 0.f;
      }
      load_g(r + 1 < nrows ? i0 + r + 1 : i0);
      const long long tk0 = p.trace ? clock64() : 0;
      int k0 = 0;
      for (; k0 + KS <= n; k0 += KS) {
        mbar_wait(&full[slot], phase);
        const VT* sb = reinterpret_cast<const VT*>(ring + (size_t)slot * slot_floats);
        if (p.pre) {   // NEXT-1: the slot holds S_ij (n = KS = 1)
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            const float4 c = sb[q * nkt + kt];
            s[q][0] = c.x;
            s[q][1] = c.y;
            s[q][2] = c.z;
            s[q][3] = c.w;
          }
        } else if (!(p.diag & COT_DIAG_NO_COMPUTE)) {
#pragma unroll
          for (int q2 = 0; q2 < KS; ++q2) {
#pragma unroll
            for (int q = 0; q < CPT; ++q) {
              const float4 c = sb[q2 * mv + q * nkt + kt];
              s[q][0] += ex2(fmaf(-c.x, c2, gc[q][0]));
              s[q][1] += ex2(fmaf(-c.y, c2, gc[q][1]));
              s[q][2] += ex2(fmaf(-c.z, c2, gc[q][2]));
              s[q][3] += ex2(fmaf(-c.w, c2, gc[q][3]));
            }
          }
        }
        release();
      }
      if (k0 < n) {   // ragged last slot of the row (n % KS != 0)
        const int kk = n - k0;
        mbar_wait(&full[slot], phase);
        const VT* sb = reinterpret_cast<const VT*>(ring + (size_t)slot * slot_floats);
        if (!(p.diag & COT_DIAG_NO_COMPUTE)) {
          for (int q2 = 0; q2 < kk; ++q2) {
#pragma unroll
            for (int q = 0; q < CPT; ++q) {
              const float4 c = sb[q2 * mv + q * nkt + kt];
              s[q][0] += ex2(fmaf(-c.x, c2, gc[q][0]));
              s[q][1] += ex2(fmaf(-c.y, c2, gc[q][1]));
              s[q][2] += ex2(fmaf(-c.z, c2, gc[q][2]));
              s[q][3] += ex2(fmaf(-c.w, c2, gc[q][3]));
            }
          }
        }
        release();
      }
      if (p.trace) c_ksum += clock64() - tk0;
      // ---- hand the row's k-sums to the epilogue warps through the queue
      mbar_wait(&qempty[qs], qph ^ 1u);
      VT* qrow = reinterpret_cast<VT*>(queue + (size_t)qs * m);
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const int jv = q * nkt + kt;
        if (jv < mv) qrow[jv] = make_float4(s[q][0], s[q][1], s[q][2], s[q][3]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&qfull[qs]);
      if (++qs == (uint32_t)QN) {
        qs = 0;
        qph ^= 1u;
      }
      ++produced;
      if (kt == 0) *(volatile unsigned*)&ctl[6] = produced;
    }
    if (p.trace && kt == 0) p.trace[blockIdx.x * 8 + 3] = c_ksum;
    asm volatile("bar.sync 3, %0;" ::"r"(nkt) : "memory");
    if (kt == 0) {
      __threadfence_block();
      *(volatile unsigned*)&ctl[7] = 1u;
      *(volatile unsigned*)&ctl[2] = 1u;     // stop the producer
    }
    // ---- drain the TMA ring: consume whatever the producer already issued
    while (true) {
      const unsigned done = lds_volatile(&ctl[1]);
      __threadfence_block();
      const unsigned iss = lds_volatile(&ctl[0]);
      if (consumed < iss) {
        mbar_wait(&full[slot], phase);
        release();
      } else if (done) {
        if (consumed >= lds_volatile(&ctl[0])) break;
      }
    }
  } else {
    // ===================================================================== epilogue warps
    // Per row (in order): wait for its k-sums in the queue and, at the first row of an iteration, for the
    // previous q-update; then the fp64 epilogue: x_ij = z_hat_j - G_ij/eps, r_i = sum_j s_ij exp(x_ij - M'_i)
    // and M_i = max_j x_ij in ONE block reduction against the previous row maximum M'_i (exact exponent
    // split), w_hat_i = log alpha_i - M'_i - log r_i (lazily, once per iteration), P_j += (alpha_i/r_i) t_ij.
    const int et = threadIdx.x - nkt;
    const int ewarp = warp - nk;
    uint32_t qs = 0, qph = 0;
    unsigned consumed = 0;
    int rbuf = 0;
    long long c_epi = 0, c_wait = 0;
    for (int r = et; r < nrows; r += net) {
      const double a = p.alpha[p.row_begin + i0 + r];
      rowstat[r * 4 + 0] = __longlong_as_double(0x7ff8000000000000LL);   // no previous maximum yet
      rowstat[r * 4 + 3] = log(a);
    }
    asm volatile("bar.sync 1, %0;" ::"r"(net) : "memory");
    double z[EPT][VEC], P[EPT][VEC];
    auto load_z = [&]() {
#pragma unroll
      for (int q = 0; q < EPT; ++q) {
        const int jv = q * net + et;
#pragma unroll
        for (int v = 0; v < VEC; ++v) z[q][v] = jv < mv ? __ldcg(p.z_hat + VEC * jv + v) : 0.0;
      }
    };
#pragma unroll
    for (int q = 0; q < EPT; ++q)
#pragma unroll
      for (int v = 0; v < VEC; ++v) P[q][v] = 0.0;
    bool halted = false;
    if (active0) load_z();
    for (int t = 0; active0 && t < p.iters && !halted; ++t) {
      if (t > 0) {   // z generation >= t: the q-update of iteration t-1 is visible
        const long long tw0 = p.trace ? clock64() : 0;
        if (et == 0) {
          unsigned zg = lds_acquire(&ctl[4]), h = lds_acquire(&ctl[5]);
          while (zg < (unsigned)t && !h) {
            __nanosleep(32);
            zg = lds_acquire(&ctl[4]);
            h = lds_acquire(&ctl[5]);
          }
          ctl[9] = h ? 1u : 0u;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(net) : "memory");
        halted = ctl[9] != 0;
        asm volatile("bar.sync 1, %0;" ::"r"(net) : "memory");
        if (p.trace) c_wait += clock64() - tw0;
        if (halted) break;
        load_z();
      }
      for (int r = 0; r < nrows; ++r) {
        // G row (read-only) first, so its latency overlaps the queue wait
        float g[EPT][VEC];
#pragma unroll
        for (int q = 0; q < EPT; ++q) {
          const int jv = q * net + et;
          const float4 gv = jv < mv ? __ldg(reinterpret_cast<const VT*>(p.G + (size_t)(i0 + r) * m) + jv)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
          g[q][0] = gv.x;
          g[q][1] = gv.y;
          g[q][2] = gv.z;
          g[q][3] = gv.w;
        }
        mbar_wait(&qfull[qs], qph);
        const long long te0 = p.trace ? clock64() : 0;
        float s[EPT][VEC];
        const VT* qrow = reinterpret_cast<const VT*>(queue + (size_t)qs * m);
#pragma unroll
        for (int q = 0; q < EPT; ++q) {
          const int jv = q * net + et;
          const float4 sv = jv < mv ? qrow[jv] : make_float4(0.f, 0.f, 0.f, 0.f);
          s[q][0] = sv.x;
          s[q][1] = sv.y;
          s[q][2] = sv.z;
          s[q][3] = sv.w;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&qempty[qs]);
        ++consumed;
        if (++qs == (uint32_t)QN) {
          qs = 0;
          qph ^= 1u;
        }
        // ---- the row epilogue
        double x[EPT][VEC];
        double lmax = -INFINITY;
#pragma unroll
        for (int q = 0; q < EPT; ++q) {
          const bool ok = q * net + et < mv;
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            x[q][v] = ok ? z[q][v] - (double)g[q][v] * inv_eps : -INFINITY;
            lmax = fmax(lmax, x[q][v]);
          }
        }
        double Mref = rowstat[r * 4 + 0];
        double tt[EPT][VEC];
        double Mtrue, rsum;
        bool exact = !(Mref == Mref);          // no previous maximum: two-pass
        if (!exact) {
          double lsum = 0.0;
#pragma unroll
          for (int q = 0; q < EPT; ++q)
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
              tt[q][v] = (x[q][v] == -INFINITY) ? 0.0 : (double)s[q][v] * exp_split(x[q][v] - Mref);
              lsum += tt[q][v];
            }
          Mtrue = lmax;
          rsum = lsum;
          cblk_maxsum(Mtrue, rsum, red2, rbuf, net, nk);
          exact = !(fabs(Mtrue - Mref) < 500.0);   // shifted sum out of the safe fp64 range: redo exactly
        } else {
          Mtrue = cblk_max1(lmax, red2, rbuf, net, nk);
        }
        if (exact) {
          Mref = Mtrue;
          double lsum = 0.0;
#pragma unroll
          for (int q = 0; q < EPT; ++q)
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
              tt[q][v] = (x[q][v] == -INFINITY) ? 0.0 : (double)s[q][v] * exp_split(x[q][v] - Mref);
              lsum += tt[q][v];
            }
          rsum = cblk_sum1(lsum, red2, rbuf, net, nk);
        }
        double rinv = (double)__frcp_rn((float)rsum);   // alpha_i / r_i: fast reciprocal + 2 Newton steps
        rinv = rinv * fma(-rsum, rinv, 2.0);
        rinv = rinv * fma(-rsum, rinv, 2.0);
        const double rho = p.alpha[p.row_begin + i0 + r] * rinv;
        if (et == 0) {
          rowstat[r * 4 + 0] = Mtrue;           // reference for the next iteration
          rowstat[r * 4 + 1] = Mref;            // shift used for r_i
          rowstat[r * 4 + 2] = rsum;
        }
#pragma unroll
        for (int q = 0; q < EPT; ++q)
#pragma unroll
          for (int v = 0; v < VEC; ++v) P[q][v] = fma(rho, tt[q][v], P[q][v]);
        if (p.trace) c_epi += clock64() - te0;
      }
      // ---- publish iteration t: w_hat of this CTA's rows (parallel logs) and the column partial
      asm volatile("bar.sync 1, %0;" ::"r"(net) : "memory");
      for (int r = et; r < nrows; r += net)
        p.w_hat[p.row_begin + i0 + r] = rowstat[r * 4 + 3] - rowstat[r * 4 + 1] - log(rowstat[r * 4 + 2]);
#pragma unroll
      for (int q = 0; q < EPT; ++q) {
        const int jv = q * net + et;
        if (jv < mv)
          reinterpret_cast<double4*>(p.partials + (size_t)u * m)[jv] =
              make_double4(P[q][0], P[q][1], P[q][2], P[q][3]);
#pragma unroll
        for (int v = 0; v < VEC; ++v) P[q][v] = 0.0;
      }
      if (p.rows_only) break;
      handoff_arrive(net + 32);               // to the sync warp (orders these writes before its B1)
    }
    if (p.trace && et == 0) {
      p.trace[blockIdx.x * 8 + 4] = c_epi;
      p.trace[blockIdx.x * 8 + 5] = c_wait;
    }
    // ---- drain the queue after a halt: consume every row the k-sum warps still produce
    (void)ewarp;
    while (true) {
      const unsigned done = lds_volatile(&ctl[7]);
      __threadfence_block();
      const unsigned prod = lds_volatile(&ctl[6]);
      if (consumed < prod) {
        mbar_wait(&qfull[qs], qph);
        __syncwarp();
        if (lane == 0) mbar_arrive(&qempty[qs]);
        ++consumed;
        if (++qs == (uint32_t)QN) {
          qs = 0;
          qph ^= 1u;
        }
      } else if (done) {
        if (consumed >= lds_volatile(&ctl[6])) break;
      }
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------------------------------------ launcher
bool tma_eligible(const IterArgs& a) {
  return a.dtype == COT_F32 && a.B == 1 && a.m % 4 == 0 && a.m <= 1024 && !(a.flags & COT_FORCE_LDG);
}

cudaError_t launch_iter_tma(const IterArgs& a, const Workspace& ws, int iters, bool rows_only, int parity,
                            cudaStream_t s) {
  const int sms = device_sm_count();
  TmaParams p;
  p.C = static_cast<const float*>(a.C);
  p.G = static_cast<const float*>(a.G);
  p.alpha = a.alpha;
  p.beta = a.beta;
  p.w_hat = a.w_hat;
  p.z_hat = a.z_hat;
  p.eps = a.eps;
  p.n = (int)a.n;
  p.m = (int)a.m;
  p.R = (int)a.R;
  p.row_begin = (int)a.row_begin;
  const UnitPlan up = unit_plan(1, a.R, sms);
  p.rpu = (int)up.rpu;
  p.U = (int)up.U;
  // ---- warp roles: k-sum warps (4 columns x CPT per thread, <= 8 warps), epilogue warps (4 x EPT)
  const int m = (int)a.m, mv = m / 4;
  int cpt = 1;
  while ((mv + 32 * cpt - 1) / (32 * cpt) > 8) cpt *= 2;
  p.nk = (mv + 32 * cpt - 1) / (32 * cpt);
  p.ne = std::max(std::max(1, p.nk / 2), (mv + 63) / 64);   // <= 2 float4 per epilogue thread
  if (const char* ev = getenv("COT_NE")) p.ne = std::max(1, std::min(8, atoi(ev)));   // tuning experiments
  int ept = 1;
  while ((mv + 32 * p.ne - 1) / (32 * p.ne) > ept) ept *= 2;
  if (cpt > 1 || ept > 2) return cudaErrorInvalidValue;
  // ---- TMA ring and row queue
  const int row_bytes = m * 4;
  int KS = 1;
  int ks_bytes = 65536;
  if (const char* ev = getenv("COT_SLOT_BYTES")) ks_bytes = atoi(ev);   // tuning experiments
  while (KS * 2 <= 16 && KS * 2 * row_bytes <= ks_bytes && KS * 2 <= (int)a.n) KS *= 2;
  p.KS = KS;
  const size_t slot_bytes = (size_t)p.KS * row_bytes;
  p.qn = std::max(1, std::min(p.rpu, 8));
  if (const char* ev = getenv("COT_QN")) p.qn = std::max(1, atoi(ev));
  const size_t queue_bytes = (size_t)p.qn * row_bytes + (size_t)p.rpu * 4 * 8;
  const size_t budget = 220 * 1024;
  if (queue_bytes + 2 * slot_bytes + 4096 > budget) return cudaErrorInvalidConfiguration;
  p.nslot = (int)std::max<size_t>(2, std::min<size_t>(64, (budget - queue_bytes - 4096) / slot_bytes));
  // ring + 1 KiB pad (branch-free over-reads past the last column stay in-bounds) + row queue + row
  // statistics + barriers + control + reduction scratch
  const size_t smem = (size_t)p.nslot * slot_bytes + 1024 + queue_bytes + ((size_t)p.nslot + p.qn) * 16 + 64 +
                      128 * 8 + 64;
  p.iters = rows_only ? 1 : iters;
  p.rows_only = rows_only ? 1 : 0;
  p.tol = a.tol;
  p.check_every = a.check_every > 0 ? a.check_every : 1;
  p.partials = ws.partials[rows_only ? (parity & 1) : 0];
  p.resid_part = ws.resid_part;
  p.state = ws.state;
  p.bar = ws.grid_bar;
  p.evict_last_rows = 0;
  p.diag = (int)(a.flags & (COT_DIAG_NO_COMPUTE | COT_DIAG_NO_SYNC));
  p.pre = (a.flags & COT_PRECOMPUTED) ? 1 : 0;
  if (const char* ev = getenv("COT_EVICT_LAST_ROWS")) p.evict_last_rows = atoi(ev);   // L2 residency experiment
  p.trace = nullptr;
  static unsigned long long* trace_buf = nullptr;   // diagnostics only (COT_TRACE=1)
  if (getenv("COT_TRACE")) {
    if (!trace_buf) cudaMalloc(&trace_buf, 4096 * 8 * sizeof(unsigned long long));
    cudaMemsetAsync(trace_buf, 0, 4096 * 8 * sizeof(unsigned long long), s);
    p.trace = trace_buf;
  }
  const int threads = (p.nk + p.ne + 2) * 32;
  cudaError_t e;
  void* fn = nullptr;
#define COT_PICK(C_, E_, K_) \
  if (cpt == C_ && ept == E_ && KS == K_) fn = (void*)k_iter_tma<C_, E_, K_>;
#define COT_PICK_K(C_, E_) \
  COT_PICK(C_, E_, 1) COT_PICK(C_, E_, 2) COT_PICK(C_, E_, 4) COT_PICK(C_, E_, 8) COT_PICK(C_, E_, 16)
  COT_PICK_K(1, 1) COT_PICK_K(1, 2)
#undef COT_PICK_K
#undef COT_PICK
  if (!fn) return cudaErrorInvalidValue;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  if (up.U > (int64_t)occ * sms) return cudaErrorInvalidConfiguration;   // one unit per co-resident CTA
  const int grid = (int)up.U;
  void* args[] = {&p};
  if (rows_only) return cudaLaunchKernel(fn, dim3(grid), dim3(threads), args, smem, s);
  e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(threads), args, smem, s);
  if (e == cudaSuccess && p.trace) {   // diagnostics: print cycle breakdown (averaged over CTAs)
    std::vector<unsigned long long> h((size_t)grid * 8);
    cudaStreamSynchronize(s);
    cudaMemcpy(h.data(), p.trace, h.size() * 8, cudaMemcpyDeviceToHost);
    double acc[8] = {0}, mx[8] = {0};
    for (int b = 0; b < grid; ++b)
      for (int k = 0; k < 8; ++k) {
        acc[k] += (double)h[(size_t)b * 8 + k] / grid;
        mx[k] = std::max(mx[k], (double)h[(size_t)b * 8 + k]);
      }
    const double it = iters > 0 ? iters : 1;
    fprintf(stderr,
            "[cot trace] iters=%d per-iter cycles (mean/max over CTAs): prod_wait %.0f/%.0f prod_total %.0f/%.0f "
            "ksum %.0f/%.0f epi_busy %.0f/%.0f epi_wait_z %.0f/%.0f\n",
            iters, acc[0] / it, mx[0] / it, acc[1] / it, mx[1] / it, acc[3] / it, mx[3] / it, acc[4] / it,
            mx[4] / it, acc[5] / it, mx[5] / it);
  }
  return e;
}

}  // namespace cot
