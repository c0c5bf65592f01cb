// K-ITER (TMA path): a persistent, warp-specialised cyclic Sinkhorn kernel for one problem (B == 1) with
// fp32 costs and m % 4 == 0. Same arithmetic as k_rows_ldg + k_cols (k_iter.cu), organised for HBM:
//
//   producer warp (1 elected lane): streams the rows of C owned by this CTA through an NSLOT-deep ring of
//     shared-memory slots with 1-D TMA bulk copies (cp.async.bulk, SASS UBLKCP); each slot holds KS
//     consecutive k-rows C[k][i][0..m) of one row i; completion is tracked by mbarrier transaction
//     counts (full[]), reuse by consumer-warp arrivals (empty[]). The producer does not depend on the
//     potentials, so it runs ahead across row epilogues, grid barriers and iteration boundaries.
//   consumer warps: per row, s_ij = sum_k exp2((G_ij - C_ijk) * log2e/eps) from the slots (one FFMA + one
//     MUFU.EX2 + one FADD per element), then the fp64 row epilogue (M_i, r_i, w_hat_i, column partials).
//     After all rows: device-wide barrier; each CTA reduces its slice of columns over all units in a fixed
//     order (deterministic), updates z_hat (q-update) and its monitor partial; device-wide barrier; every
//     CTA sums the monitor partials in the same order and applies the same freeze rule.
//
// The grid is co-resident (cooperative launch, one CTA per SM), which the device-wide barrier requires.
// With rows_only = 1 the kernel performs only the row pass of one iteration (no barriers): cerot_rows.
#include "common.cuh"
#include "internal.h"

#include <algorithm>

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
  unsigned* bar;         // [2]: device-wide barrier arrival count, generation
  int evict_last_rows;   // rows [0, evict_last_rows) of every block are streamed with an L2 evict_last hint
};

__device__ __forceinline__ void cbar(int nthreads) {   // consumer-only named barrier
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}
__device__ __forceinline__ unsigned ld_volatile(const unsigned* p) {
  unsigned v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned lds_volatile(const unsigned* p) { return *(volatile const unsigned*)p; }

// Device-wide barrier among the consumer warps of all CTAs, split into arrive / wait so that independent
// work can run in between. bar = {arrival count, generation}; arrive returns the generation to wait past.
__device__ __forceinline__ unsigned grid_arrive(unsigned* bar, int nct) {
  __shared__ unsigned gen_sh;
  cbar(nct);
  if (threadIdx.x == 0) {
    const unsigned gen = ld_volatile(bar + 1);
    __threadfence();
    const unsigned arrived = atomicAdd(bar, 1u);
    if (arrived == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    }
    gen_sh = gen;
  }
  cbar(nct);
  return gen_sh;
}
__device__ __forceinline__ void grid_wait(unsigned* bar, unsigned gen, int nct) {
  if (threadIdx.x == 0) {
    while (ld_volatile(bar + 1) == gen) __nanosleep(20);
    __threadfence();
  }
  cbar(nct);
}
__device__ __forceinline__ void grid_barrier(unsigned* bar, int nct) { grid_wait(bar, grid_arrive(bar, nct), nct); }

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
__device__ __forceinline__ double cblk_max(double v, double* sh, int nct) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_max(v);
  if (lane == 0) sh[wid] = v;
  cbar(nct);
  double t = sh[0];
  for (int w = 1; w < (nct >> 5); ++w) t = fmax(t, sh[w]);
  cbar(nct);
  return t;
}

template <int CPT, int KS>
__global__ void __launch_bounds__(288, 1) k_iter_tma(TmaParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int nwarps = blockDim.x >> 5;
  const int ncw = nwarps - 1;                 // consumer warps; the last warp produces
  const int nct = ncw * 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = p.m, mv = m >> 2;
  const size_t slot_floats = (size_t)KS * m;
  float* ring = reinterpret_cast<float*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)p.nslot * slot_floats * 4 + 1024);
  uint64_t* empty = full + p.nslot;
  unsigned* ctl = reinterpret_cast<unsigned*>(empty + p.nslot);   // [0] issued, [1] producer done, [2] stop
  double* red = reinterpret_cast<double*>(ctl + 4);               // 32 doubles

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.nslot; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], ncw);
    }
    ctl[0] = 0;
    ctl[1] = 0;
    ctl[2] = 0;
    fence_mbar_init();
  }
  __syncthreads();

  const int n = p.n, R = p.R;
  const int U = p.U, rpu = p.rpu;

  if (warp == ncw) {
    // ===================================================================== producer (one lane)
    if (lane == 0) {
      const uint64_t pol_first = policy_evict_first();
      const uint64_t pol_last = policy_evict_last();
      uint32_t slot = 0, phase = 0;
      unsigned issued = 0;
      const uint32_t row_bytes = (uint32_t)m * 4u;
      for (int t = 0; t < p.iters; ++t) {
        for (int u = blockIdx.x; u < U; u += gridDim.x) {
          const int i0 = u * rpu, i1 = min(R, i0 + rpu);
          for (int i = i0; i < i1; ++i) {
            const uint64_t pol = i < p.evict_last_rows ? pol_last : pol_first;
            for (int k0 = 0; k0 < n; k0 += KS) {
              if (lds_volatile(&ctl[2])) goto producer_done;
              const int kk = min(KS, n - k0);
              mbar_wait(&empty[slot], phase ^ 1u);
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
      }
    producer_done:
      __threadfence_block();
      *(volatile unsigned*)&ctl[1] = 1u;
    }
    __syncwarp();
  } else {
    // ===================================================================== consumers
    const int ct = threadIdx.x;
    const double inv_eps = 1.0 / p.eps[0];
    const float c2 = (float)(COT_LOG2E * inv_eps);
    uint32_t slot = 0, phase = 0;
    unsigned consumed = 0;
    SolverState st = p.state[0];
    bool active = st.active != 0;
    const int cols_per_cta = (m + gridDim.x - 1) / gridDim.x;
    const int col0 = blockIdx.x * cols_per_cta;
    const int col1 = min(m, col0 + cols_per_cta);
    bool pending = false;       // a q-update barrier whose wait is deferred to the next epilogue
    unsigned pending_gen = 0;
    for (int t = 0; t < p.iters && active; ++t) {
      for (int u = blockIdx.x; u < U; u += gridDim.x) {
        const int i0 = u * rpu, i1 = min(R, i0 + rpu);
        double z[CPT][4], P[CPT][4];
        float4 gnext[CPT];
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
          const int jv = q * nct + ct;
          const bool ok = jv < mv;
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            z[q][v] = (ok && !pending) ? __ldcg(p.z_hat + 4 * jv + v) : 0.0;
            P[q][v] = 0.0;
          }
          gnext[q] = ok ? __ldg(reinterpret_cast<const float4*>(p.G + (size_t)i0 * m) + jv) : make_float4(0, 0, 0, 0);
        }
        for (int i = i0; i < i1; ++i) {
          float g[CPT][4], gc[CPT][4], s[CPT][4];
          const bool first_row = (i == i0) && (u == (int)blockIdx.x);
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            g[q][0] = gnext[q].x;
            g[q][1] = gnext[q].y;
            g[q][2] = gnext[q].z;
            g[q][3] = gnext[q].w;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              gc[q][v] = g[q][v] * c2;
              s[q][v] = 0.f;
            }
            const int jv = q * nct + ct;
            if (i + 1 < i1 && jv < mv) gnext[q] = __ldg(reinterpret_cast<const float4*>(p.G + (size_t)(i + 1) * m) + jv);
          }
          // ---- the streamed k-sum over this row's slots. Threads past the last column read (in-bounds)
          //      smem garbage that the epilogue masks out, so the body has no per-column branches.
          int k0 = 0;
          for (; k0 + KS <= n; k0 += KS) {
            mbar_wait(&full[slot], phase);
            const float4* sb = reinterpret_cast<const float4*>(ring + (size_t)slot * slot_floats);
#pragma unroll
            for (int q2 = 0; q2 < KS; ++q2) {
#pragma unroll
              for (int q = 0; q < CPT; ++q) {
                const float4 c = sb[q2 * mv + q * nct + ct];
                s[q][0] += ex2(fmaf(-c.x, c2, gc[q][0]));
                s[q][1] += ex2(fmaf(-c.y, c2, gc[q][1]));
                s[q][2] += ex2(fmaf(-c.z, c2, gc[q][2]));
                s[q][3] += ex2(fmaf(-c.w, c2, gc[q][3]));
              }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            ++consumed;
            if (++slot == (uint32_t)p.nslot) {
              slot = 0;
              phase ^= 1u;
            }
          }
          if (k0 < n) {   // ragged last slot of the row (n % KS != 0)
            const int kk = n - k0;
            mbar_wait(&full[slot], phase);
            const float4* sb = reinterpret_cast<const float4*>(ring + (size_t)slot * slot_floats);
            for (int q2 = 0; q2 < kk; ++q2) {
#pragma unroll
              for (int q = 0; q < CPT; ++q) {
                const float4 c = sb[q2 * mv + q * nct + ct];
                s[q][0] += ex2(fmaf(-c.x, c2, gc[q][0]));
                s[q][1] += ex2(fmaf(-c.y, c2, gc[q][1]));
                s[q][2] += ex2(fmaf(-c.z, c2, gc[q][2]));
                s[q][3] += ex2(fmaf(-c.w, c2, gc[q][3]));
              }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            ++consumed;
            if (++slot == (uint32_t)p.nslot) {
              slot = 0;
              phase ^= 1u;
            }
          }
          // ---- fp64 row epilogue (needs z_hat of the previous q-update: wait for that barrier here,
          //      after this row's k-sum, which does not depend on z)
          if (first_row && pending) {
            grid_wait(p.bar + 2, pending_gen, nct);
            pending = false;
#pragma unroll
            for (int q = 0; q < CPT; ++q) {
              const int jv = q * nct + ct;
#pragma unroll
              for (int v = 0; v < 4; ++v) z[q][v] = jv < mv ? __ldcg(p.z_hat + 4 * jv + v) : 0.0;
            }
          }
          double x[CPT][4];
          double lmax = -INFINITY;
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            const bool ok = q * nct + ct < mv;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              x[q][v] = ok ? z[q][v] - (double)g[q][v] * inv_eps : -INFINITY;
              lmax = fmax(lmax, x[q][v]);
            }
          }
          const double M = cblk_max(lmax, red, nct);
          double tt[CPT][4];
          double lsum = 0.0;
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            const bool ok = q * nct + ct < mv;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const double e = (double)ex2((float)((x[q][v] - M) * COT_LOG2E));
              tt[q][v] = ok ? (double)s[q][v] * e : 0.0;
              lsum += tt[q][v];
            }
          }
          const double r = cblk_sum(lsum, red, nct);
          const double a = p.alpha[p.row_begin + i];
          if (ct == 0) p.w_hat[p.row_begin + i] = log(a) - M - log(r);
          const double rho = a / r;
#pragma unroll
          for (int q = 0; q < CPT; ++q)
#pragma unroll
            for (int v = 0; v < 4; ++v) P[q][v] = fma(rho, tt[q][v], P[q][v]);
        }
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
          const int jv = q * nct + ct;
          if (jv < mv)
            reinterpret_cast<double4*>(p.partials + (size_t)u * m)[jv] = make_double4(P[q][0], P[q][1], P[q][2], P[q][3]);
        }
      }
      if (p.rows_only) break;
      // ---- column pass over this CTA's column slice (fixed order => deterministic)
      grid_barrier(p.bar, nct);
      double dev = 0.0;
      for (int j = col0 + warp; j < col1; j += ncw) {
        double acc = 0.0;
        for (int u = lane; u < U; u += 32) acc += __ldcg(p.partials + (size_t)u * m + j);
        acc = warp_sum(acc);
        if (lane == 0) {
          const double bj = p.beta[j];
          dev += fabs(acc - bj);
          if (!(acc >= 1e-28)) atomicOr(&p.state[0].flags, (int)STATE_UNDERFLOW);
          p.z_hat[j] = __ldcg(p.z_hat + j) + (log(bj) - log(acc));
        }
      }
      // the monitor is needed at check iterations (freeze rule) and after the last iteration (report)
      const bool need_resid = (p.tol > 0.0 && (st.iters + 1) % p.check_every == 0) || (t == p.iters - 1);
      if (need_resid) {
        dev = cblk_sum(dev, red, nct);
        if (ct == 0) p.resid_part[blockIdx.x] = dev;
        grid_barrier(p.bar + 2, nct);
        if (warp == 0) {
          double r = 0.0;
          for (int b2 = lane; b2 < (int)gridDim.x; b2 += 32) r += __ldcg(p.resid_part + b2);
          r = warp_sum(r);
          if (lane == 0) red[0] = r * (double)n;
        }
        cbar(nct);
        st.residual = red[0];
        cbar(nct);
      } else {
        pending_gen = grid_arrive(p.bar + 2, nct);
        pending = true;
      }
      st.iters += 1;
      if (p.tol > 0.0 && st.iters % p.check_every == 0 && st.residual <= p.tol) {
        st.active = 0;
        st.converged = 1;
        active = false;
      }
    }
    if (pending) grid_wait(p.bar + 2, pending_gen, nct);
    if (blockIdx.x == 0 && ct == 0 && !p.rows_only) {
      SolverState out = p.state[0];
      out.iters = st.iters;
      out.residual = st.residual;
      out.active = st.active;
      out.converged = st.converged;
      p.state[0] = out;
    }
    // ---- drain: stop the producer and consume whatever it already issued
    if (ct == 0) *(volatile unsigned*)&ctl[2] = 1u;
    cbar(nct);
    while (true) {
      const unsigned done = lds_volatile(&ctl[1]);
      __threadfence_block();
      const unsigned iss = lds_volatile(&ctl[0]);
      if (consumed < iss) {
        mbar_wait(&full[slot], phase);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        ++consumed;
        if (++slot == (uint32_t)p.nslot) {
          slot = 0;
          phase ^= 1u;
        }
      } else if (done) {
        if (consumed >= lds_volatile(&ctl[0])) break;
      }
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------------------------------------ launcher
bool tma_eligible(const IterArgs& a) {
  return a.dtype == COT_F32 && a.B == 1 && a.m % 4 == 0 && a.m <= 4096 && !(a.flags & COT_FORCE_LDG);
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
  const int row_bytes = (int)a.m * 4;
  int KS = 1;
  while (KS * 2 <= 16 && KS * 2 * row_bytes <= 16384 && KS * 2 <= (int)a.n) KS *= 2;
  p.KS = KS;
  const size_t slot_bytes = (size_t)p.KS * row_bytes;
  const size_t budget = 200 * 1024;
  p.nslot = (int)std::max<size_t>(2, std::min<size_t>(64, (budget - 2048) / slot_bytes));
  // ring + 1 KiB pad (branch-free over-reads past the last column stay in-bounds) + barriers + control
  const size_t smem = (size_t)p.nslot * slot_bytes + 1024 + (size_t)p.nslot * 16 + 16 + 32 * 8 + 64;
  p.iters = rows_only ? 1 : iters;
  p.rows_only = rows_only ? 1 : 0;
  p.tol = a.tol;
  p.check_every = a.check_every > 0 ? a.check_every : 1;
  p.partials = ws.partials[rows_only ? (parity & 1) : 0];
  p.resid_part = ws.resid_part;
  p.state = ws.state;
  p.bar = ws.grid_bar;
  p.evict_last_rows = 0;
  const int mv = (int)a.m / 4;
  int ncw = (mv + 31) / 32;
  int cpt = 1;
  while (ncw > 8) {
    cpt *= 2;
    ncw = (mv / cpt + 31) / 32;
  }
  const int threads = (ncw + 1) * 32;
  cudaError_t e;
  void* fn = nullptr;
#define COT_PICK(C_, K_) \
  if (cpt == C_ && KS == K_) fn = (void*)k_iter_tma<C_, K_>;
  COT_PICK(1, 1) COT_PICK(1, 2) COT_PICK(1, 4) COT_PICK(1, 8) COT_PICK(1, 16)
  COT_PICK(2, 1) COT_PICK(2, 2) COT_PICK(2, 4) COT_PICK(2, 8) COT_PICK(2, 16)
  COT_PICK(4, 1) COT_PICK(4, 2) COT_PICK(4, 4) COT_PICK(4, 8) COT_PICK(4, 16)
#undef COT_PICK
  if (!fn) return cudaErrorInvalidValue;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  const int grid = (int)std::min<int64_t>(up.U, (int64_t)occ * sms);
  void* args[] = {&p};
  if (rows_only) return cudaLaunchKernel(fn, dim3(grid), dim3(threads), args, smem, s);
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(threads), args, smem, s);
}

}  // namespace cot
