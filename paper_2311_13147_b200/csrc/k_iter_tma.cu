// K-ITER (TMA path): a persistent, warp-specialised cyclic Sinkhorn kernel for one problem (B == 1) with
// fp32 costs and m % 4 == 0 (Alg. 2 lines 4-5, in the log domain of eq. P:403-411). Same arithmetic
// as k_rows_ldg + k_cols (k_iter.cu), organised for HBM. One CTA per SM owns a unit of consecutive rows;
// three warp roles:
//
//   producer warp (1 elected lane): streams the CTA's rows of C through an NSLOT-deep ring of shared-
//     memory slots with 1-D TMA bulk copies (cp.async.bulk, SASS UBLKCP); a slot holds KS consecutive
//     k-rows C[k][i][0..m) of one row i; completion via mbarrier transaction counts (full[]), reuse via
//     consumer-warp arrivals (empty[]). It never depends on the potentials, so it runs ahead across
//     epilogues, device-wide steps and iteration boundaries.
//   k-sum warps: s_ij = sum_k exp2((G_ij - C_ijk) * log2e/eps) (one FFMA + one MUFU.EX2 + one FADD per
//     element) into a shared-memory row queue; s is iterate-independent, so they run up to a queue ahead.
//   epilogue warps: rows in batches of RB with one block reduction per batch: x_ij = z_hat_j - G_ij/eps
//     (-G/eps staged in fp64 shared memory), t_ij = s_ij exp(x_ij - M'_i) against the row's log-sum-exp of the
//     previous iteration (exact exponent split; a batch out of range is redone exactly), r_i, w_hat_i,
//     P_j += (alpha_i / r_i) t_ij; then the device-wide steps WITHOUT a grid barrier: the CTA's partial is
//     published as LL lines (16-byte stores carrying the iteration's generation), the owner of each column
//     slice polls the slice's lines of every unit and sums them in unit order (deterministic), [fused
//     multi-GPU: exchanges the slice sums with every rank through peer-mapped LL lines, summed in rank order],
//     applies the q-update z_hat_j += log beta_j - log c_j and publishes z_hat as LL lines, which every CTA
//     polls before its next iteration; the monitor is one LL line per slice owner.
//
// The grid is co-resident (cooperative launch). With rows_only = 1 the kernel performs only the row pass
// of one iteration into plain fp64 partials (no device-wide steps): cerot_rows / cerot_rows_shard.
#include "common.cuh"
#include "internal.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
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
  double* partials;      // [U][m] (rows_only: the plain fp64 column partials of cerot_rows)
  SolverState* state;    // [1]
  // device-wide steps through LL lines (workspace; zeroed by cerot_init): generation g = lepoch + iteration
  uint4* plines;         // [2][lcap][m] column partials of each unit
  uint4* zlines;         // [m] z_hat after the q-update
  uint4* rlines;         // [2][lcap] monitor partial of each column slice
  unsigned long long* lepoch;   // iterations run on this workspace since cerot_init
  int lcap;              // unit capacity of the line arrays (>= U)
  int gsh;               // 1: this CTA's rows of G are staged in shared memory
  int nk, ne, qn;        // k-sum warps, epilogue warps, row-queue depth
  int evict_last_rows;   // rows [0, evict_last_rows) of every block are streamed with an L2 evict_last hint
  int diag;              // COT_DIAG_* bits (diagnostics only)
  int pre;               // precomputed mode (NEXT-1): C is S [R][m] (n = 1) and s_ij = S_ij
  int kres;              // k-blocks [0, kres) of the CTA's rows are resident in shared memory (loaded once per
                         // launch); only [kres, n) is streamed through the ring every iteration
  int ktm;               // k-blocks [kres, kres + ktm) of the CTA's rows are resident in TENSOR memory (each k-sum
                         // thread's own columns of them, loaded once per launch; a multiple of 4): the ring
                         // streams [kres + ktm, n)
  int rpw;               // row-per-warp epilogue (several rows per CTA, EPT == 1): no block reduction per row
  int det;               // deterministic mode: 128-bit fixed-point column partials (implies rpw); 2 lines per value
  unsigned long long* trace;   // diagnostics: [grid][8] cycle counters, or nullptr
  // fused multi-GPU mode (nranks > 0): the column sums of each slice are exchanged through LL lines
  int nranks, rank;      // ranks of the row partition, this rank
  int ncs;               // column slices (identical on every rank)
  uint4* xpeer[kMaxRanks];          // rank q's line array [2][nranks][m], mapped into this rank's address space
  unsigned long long* xepoch;       // this rank's exchange epoch (iterations exchanged so far)
};

__device__ __forceinline__ void cbar(int nthreads) {   // consumer-only named barrier
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}
// OR of a predicate over the `nthreads` threads of named barrier 1 (a barrier itself: every epilogue thread calls it)
__device__ __forceinline__ bool bar_red_or(bool v, int nthreads) {
  unsigned r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\tbar.red.or.pred q, 1, %2, p;\n\tselp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"((unsigned)v), "r"(nthreads)
      : "memory");
  return r != 0;
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
// LL lines of the fused multi-GPU exchange: 16-byte volatile stores / loads on (possibly peer-mapped)
// global memory; each 8-byte half {32-bit payload, 32-bit generation} is written and read as one unit.
__device__ __forceinline__ void st_line(uint4* p, uint4 v) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 ld_line(const uint4* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr unsigned long long kPeerTimeoutNs = 20000000000ull;   // 20 s without a peer's line: give up
#ifndef COT_POLL_BACKOFF_NS
#define COT_POLL_BACKOFF_NS 0
#endif
constexpr unsigned kPollBackoffNs = COT_POLL_BACKOFF_NS;
constexpr int kColScratch = 256 + 2 * kMaxRanks * 8;   // doubles: column-pass groups, then the rank exchange
constexpr int kRankScratch = 256;

__device__ __forceinline__ uint4 ll_pack(double v, unsigned g) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return make_uint4((unsigned)b, g, (unsigned)(b >> 32), g);
}
__device__ __forceinline__ bool ll_ready(const uint4& l, unsigned g) { return l.y == g && l.w == g; }
__device__ __forceinline__ double ll_value(const uint4& l) {
  return __longlong_as_double((long long)(((unsigned long long)l.z << 32) | l.x));
}
// Spin until the line carries generation g; false after kPeerTimeoutNs (v is then garbage).
__device__ __forceinline__ bool poll_line(const uint4* a, unsigned g, double& v) {
  uint4 l = ld_line(a);
  if (ll_ready(l, g)) {
    v = ll_value(l);
    return true;
  }
  const unsigned long long t0 = gtimer();
  while (true) {
    if (kPollBackoffNs) __nanosleep(kPollBackoffNs);   // fewer L2 requests while waiting
    l = ld_line(a);
    if (ll_ready(l, g)) {
      v = ll_value(l);
      return true;
    }
    if (gtimer() - t0 > kPeerTimeoutNs) {
      v = 0.0;
      return false;
    }
  }
}

// Sum (or max) of up to 8 values r[0], r[stride], ...: all loads issued first, then a fixed pairwise tree
// (one shared-memory latency instead of a chain of nw).
__device__ __forceinline__ double tree8(const double* r, int nw, bool is_max) {
  double v[8];
#pragma unroll
  for (int w = 0; w < 8; ++w) v[w] = w < nw ? r[w] : (is_max ? -INFINITY : 0.0);
#pragma unroll
  for (int h = 4; h >= 1; h >>= 1)
#pragma unroll
    for (int w = 0; w < h; ++w) v[w] = is_max ? fmax(v[w], v[w + h]) : v[w] + v[w + h];
  return v[0];
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
  mx = tree8(r, nct >> 5, true);
  sm = tree8(r + 32, nct >> 5, false);
  buf ^= 1;
}
__device__ __forceinline__ double cblk_sum1(double v, double* red2, int& buf, int nct, int wbase) {
  double m = -INFINITY;
  cblk_maxsum(m, v, red2, buf, nct, wbase);
  return v;
}

// The epilogue's exponentials in split form. Every term is t_ij = s'_ij 2^{zL_j - kM_i - a_ij} with
// s'_ij = sum_k 2^{a_ij - C_ijk log2e/eps} from the k-sum warps (a_ij = round(G_ij log2e/eps), an integer, so
// s'_ij lies in [2^-1/2, 1.42 n]), zL_j = z_j log2e and kM_i an integer row shift (the rounded log2 of the
// previous iteration's row log-sum-exp). zL_j is split once per column per iteration into an integer kz_j and
// Fz_j = 2^{zL_j - kz_j} in fp64 (split_pow2_fp64); per element that leaves an integer exponent
// e = kz_j - kM_i - a_ij assembled into the fp64 bits of s'_ij (ldexp_pos, no conversion) and one fp64
// product by Fz_j. The only per-element rounding is the fp32 k-sum's (random across i, averaged in the
// column sums); no factor common to a row or a column is rounded below fp64.
// (split_pow2_fp64 and ldexp_pos: common.cuh)

// Deterministic mode (COT_DETERMINISTIC): column partials in 128-bit unsigned fixed point with 120 fraction
// bits. Every term (alpha_i / r_i) t_ij >= 0 is truncated to a multiple of 2^-120 on its own, so the integer
// sums are exact and do not depend on how rows are grouped into CTAs or ranks.
__device__ __forceinline__ void fx_add(unsigned long long& lo, unsigned long long& hi, unsigned long long lo2,
                                       unsigned long long hi2) {
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(lo), "+l"(hi) : "l"(lo2), "l"(hi2));
}
__device__ __forceinline__ void fx_acc(double x, unsigned long long& lo, unsigned long long& hi) {   // += x 2^120
  if (!(x > 0.0)) return;
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  const int e = (int)(b >> 52) - 1075 + 120;   // x 2^120 = mant 2^e (x < 2^8 is guaranteed: e <= 75)
  const unsigned long long mant = (b & 0xFFFFFFFFFFFFFull) | (1ull << 52);
  unsigned long long l = 0, h = 0;
  if (e > 75) {   // unreachable (sum(alpha) < 2^7 is checked before the launch iterates): saturate, no UB
    l = h = ~0ull;
  } else if (e >= 64) {
    h = mant << (e - 64);
  } else if (e > 0) {
    l = mant << e;
    h = mant >> (64 - e);
  } else if (e > -64) {
    l = mant >> (-e);
  }
  fx_add(lo, hi, l, h);
}
__device__ __forceinline__ double fx_to_double(unsigned long long lo, unsigned long long hi) {
  return (double)hi * 0x1p-56 + (double)lo * 0x1p-120;
}
__device__ __forceinline__ unsigned long long dbits(double x) { return (unsigned long long)__double_as_longlong(x); }
__device__ __forceinline__ double bitsd(unsigned long long x) { return __longlong_as_double((long long)x); }

// One-barrier block reductions of N values over the epilogue warps (<= 8 warps; double-buffered scratch).
// The sums use a transposed butterfly: at the first levels each lane keeps half of its values and sends the
// other half, so N = 4 rows cost 6 double shuffles per warp instead of 20 (fixed order: deterministic).
template <int N>
__device__ __forceinline__ void cblk_sumN(double* v, double* red2, int& buf, int nct, int wbase) {
  static_assert(N == 2 || N == 4, "row batches of 2 or 4");
  const int lane = threadIdx.x & 31, wid = (threadIdx.x >> 5) - wbase;
  double* r = red2 + buf * 64;
  int row;
  double k;
  if (N == 4) {
    const bool hi = lane & 16;
    const double s0 = __shfl_xor_sync(0xffffffffu, hi ? v[0] : v[2], 16);
    const double s1 = __shfl_xor_sync(0xffffffffu, hi ? v[1] : v[3], 16);
    const double k0 = (hi ? v[2] : v[0]) + s0, k1 = (hi ? v[3] : v[1]) + s1;   // rows 2hi, 2hi+1
    const bool h8 = lane & 8;
    k = (h8 ? k1 : k0) + __shfl_xor_sync(0xffffffffu, h8 ? k0 : k1, 8);
    row = (hi ? 2 : 0) + (h8 ? 1 : 0);
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
    if ((lane & 7) == 0) r[row * 8 + wid] = k;
  } else {
    const bool hi = lane & 16;
    k = (hi ? v[1] : v[0]) + __shfl_xor_sync(0xffffffffu, hi ? v[0] : v[1], 16);
    row = hi ? 1 : 0;
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
    if ((lane & 15) == 0) r[row * 8 + wid] = k;
  }
  cbar(nct);
#pragma unroll
  for (int q = 0; q < N; ++q) v[q] = tree8(r + q * 8, nct >> 5, false);
  buf ^= 1;
}
template <int N>
__device__ __forceinline__ void cblk_maxN(double* v, double* red2, int& buf, int nct, int wbase) {
  const int lane = threadIdx.x & 31, wid = (threadIdx.x >> 5) - wbase;
  double* r = red2 + buf * 64;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const double x = warp_max(v[k]);
    if (lane == 0) r[k * 8 + wid] = x;
  }
  cbar(nct);
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = tree8(r + k * 8, nct >> 5, true);
  buf ^= 1;
}

// k-sum of four consecutive k-rows at `b` (row stride mv float4s): all loads first, then the 16 x CPT independent
// FFMA + MUFU.EX2 back to back, then a fixed pairwise sum per element (in-order issue would otherwise stall on
// each MUFU result before the next k-row's work)
template <int CPT>
__device__ __forceinline__ void ksum4(const float4* __restrict__ b, int mv, int nkt, int kt, const float c2,
                                      const float (&gc)[CPT][4], float (&s)[CPT][4]) {
  float4 c[4][CPT];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
#pragma unroll
    for (int q = 0; q < CPT; ++q) c[kk][q] = b[(size_t)kk * mv + q * nkt + kt];
  float e[4][CPT][4];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      e[kk][q][0] = ex2(fmaf(-c[kk][q].x, c2, gc[q][0]));
      e[kk][q][1] = ex2(fmaf(-c[kk][q].y, c2, gc[q][1]));
      e[kk][q][2] = ex2(fmaf(-c[kk][q].z, c2, gc[q][2]));
      e[kk][q][3] = ex2(fmaf(-c[kk][q].w, c2, gc[q][3]));
    }
#pragma unroll
  for (int q = 0; q < CPT; ++q)
#pragma unroll
    for (int v = 0; v < 4; ++v) s[q][v] += (e[0][q][v] + e[1][q][v]) + (e[2][q][v] + e[3][q][v]);
}
template <int CPT>
__device__ __forceinline__ void ksum1(const float4* __restrict__ b, int nkt, int kt, const float c2,
                                      const float (&gc)[CPT][4], float (&s)[CPT][4]) {
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    const float4 c = b[q * nkt + kt];
    s[q][0] += ex2(fmaf(-c.x, c2, gc[q][0]));
    s[q][1] += ex2(fmaf(-c.y, c2, gc[q][1]));
    s[q][2] += ex2(fmaf(-c.z, c2, gc[q][2]));
    s[q][3] += ex2(fmaf(-c.w, c2, gc[q][3]));
  }
}

template <int CPT, int EPT, int KS>
__device__ __forceinline__ void iter_tma_body(const TmaParams& p, const int bid, const int nblk) {
  constexpr int VEC = 4;
  constexpr int RS = 6;                       // rowstat stride: next reference, Mref, r, log alpha, alpha, -
  constexpr int RB = EPT == 1 ? 4 : 2;        // rows per epilogue batch
  using VT = float4;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = p.nk, ne = p.ne;             // k-sum warps, epilogue warps, then the producer warp
  const int nkt = nk * 32, net = ne * 32;
  const int wprod = nk + ne;
  const int m = p.m, mv = m / VEC;
  const int n = p.n, R = p.R;
  const int rpu = p.rpu, QN = p.qn;
  const size_t slot_floats = (size_t)KS * m;
  // ---- shared memory layout
  float* ring = reinterpret_cast<float*>(smem);
  // resident k-blocks [rpu][kres][m] after the ring and its 1 KiB over-read pad
  float* resid = reinterpret_cast<float*>(smem + (size_t)p.nslot * slot_floats * 4 + 1024);
  float* queue = resid + (size_t)rpu * p.kres * m;                                          // [QN][m]
  int* gsh = reinterpret_cast<int*>(queue + (size_t)QN * m);            // [rpu][m] a_ij = round(G_ij log2e/eps)
  double* rowstat = reinterpret_cast<double*>(gsh + (size_t)rpu * m);    // [rpu][RS] (rpu * m even: m % 4 == 0)
  double* xs = rowstat + (size_t)rpu * RS;                               // [kColScratch] column-pass scratch
  // row-per-warp mode: the column splits of z (kz, Fz) for every column and one fp64 column-partial row per
  // epilogue warp
  double* zfs = xs + kColScratch;                                          // [m] Fz_j (rpw)
  int* zks = reinterpret_cast<int*>(zfs + (p.rpw ? m : 0));               // [m] kz_j (rpw)
  double* wpart = reinterpret_cast<double*>(zks + (p.rpw ? m : 0));       // [rpu][m] row terms (rpw)
  uint64_t* full = reinterpret_cast<uint64_t*>(wpart + (p.rpw ? (size_t)rpu * m : 0));
  uint64_t* empty = full + p.nslot;
  uint64_t* qfull = empty + p.nslot;
  uint64_t* qempty = qfull + QN;
  uint64_t* resbar = qempty + QN;                                        // the resident k-blocks have landed
  unsigned* ctl = reinterpret_cast<unsigned*>(resbar + 2);
  // ctl: [0] TMA slots issued [1] producer done [2] stop producer [5] halt
  //      [6] rows produced by the k-sum warps [7] k-sum warps done [8] k-sum broadcast
  double* red2 = reinterpret_cast<double*>(ctl + 16);   // [2][64]

  const int u = bid;                        // one unit of rows per CTA (the launcher sets nblk == U)
  const int i0 = u * rpu, i1 = min(R, i0 + rpu), nrows = i1 - i0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.nslot; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nk);
    }
    for (int q = 0; q < QN; ++q) {
      mbar_init(&qfull[q], nk);
      mbar_init(&qempty[q], p.rpw ? 1 : ne);   // row-per-warp: one warp consumes a row
    }
    mbar_init(resbar, 1);
    for (int c = 0; c < 16; ++c) ctl[c] = 0;
    fence_mbar_init();
  }
  const double inv_eps = 1.0 / p.eps[0];
  const float c2 = (float)(COT_LOG2E * inv_eps);
  {   // this CTA's rows of the integer shifts a_ij, computed exactly as the k-sum warps compute them
    const VT* src = reinterpret_cast<const VT*>(p.G + (size_t)i0 * m);
    for (int idx = threadIdx.x; idx < nrows * mv; idx += blockDim.x) {
      const float4 g4 = __ldg(src + idx);
      reinterpret_cast<int4*>(gsh)[idx] = make_int4(__float2int_rn(g4.x * c2), __float2int_rn(g4.y * c2),
                                                    __float2int_rn(g4.z * c2), __float2int_rn(g4.w * c2));
    }
  }
  if (warp == 0 && p.ktm > 0) {   // all 512 TMEM columns (one CTA per SM): the TMEM-resident k-blocks
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&ctl[12])));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");

  // deterministic mode: the 128-bit fixed point (8 integer bits) holds every column partial only if
  // sum(alpha) < 2^7 (cerot_init flags larger masses); such a launch refuses to iterate (COT_E_ARG)
  const bool det_refused = p.det && (p.state[0].flags & STATE_DET_RANGE);
  const bool active0 = p.state[0].active != 0 && !det_refused;
  if (det_refused && bid == 0 && threadIdx.x == 0) atomicOr(&p.state[0].flags, (int)STATE_DET_REFUSED);

  if (warp == wprod) {
    // ===================================================================== producer (one lane)
    if (lane == 0 && active0) {
      const uint64_t pol_first = policy_evict_first();
      const uint64_t pol_last = policy_evict_last();
      if (p.kres > 0 && nrows > 0) {   // the resident k-blocks of every row of the unit, once per launch
        const uint32_t rb = (uint32_t)m * 4u;
        mbar_arrive_expect_tx(resbar, (uint32_t)nrows * (uint32_t)p.kres * rb);
        for (int i = i0; i < i1; ++i)
          for (int k = 0; k < p.kres; ++k)
            bulk_g2s(resid + ((size_t)(i - i0) * p.kres + k) * m, p.C + ((size_t)k * R + i) * m, rb, resbar,
                     pol_first);
      }
      uint32_t slot = 0, phase = 0;
      unsigned issued = 0;
      long long prod_wait = 0;
      const long long tp0 = clock64();
      const uint32_t row_bytes = (uint32_t)m * 4u;
      for (int t = 0; t < p.iters; ++t) {
        for (int i = i0; i < i1; ++i) {
          const uint64_t pol = i < p.evict_last_rows ? pol_last : pol_first;
          for (int k0 = p.kres + p.ktm; k0 < n; k0 += KS) {
            if (lds_volatile(&ctl[2])) goto producer_done;
            const int kk = min(KS, n - k0);
            const long long tw0 = p.trace ? clock64() : 0;
            mbar_wait(&empty[slot], phase ^ 1u);
            if (p.trace) prod_wait += clock64() - tw0;
            if (t > 0 && (p.diag & COT_DIAG_NO_STREAM)) {
              mbar_arrive(&full[slot]);
            } else {
              mbar_arrive_expect_tx(&full[slot], (uint32_t)kk * row_bytes);
              float* dst = ring + (size_t)slot * slot_floats;
              for (int q = 0; q < kk; ++q)
                bulk_g2s(dst + (size_t)q * m, p.C + ((size_t)(k0 + q) * R + i) * m, row_bytes, &full[slot], pol);
            }
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
        p.trace[bid * 16 + 0] = prod_wait;
        p.trace[bid * 16 + 1] = clock64() - tp0;
      }
    }
    if (lane == 0) {
      __threadfence_block();
      *(volatile unsigned*)&ctl[1] = 1u;
    }
    __syncwarp();
  } else if (warp < nk) {
    // ===================================================================== k-sum warps
    // s_ij = sum_k exp2((G_ij - C_ijk) log2e/eps) for every row, streamed from the TMA ring into the row
    // queue; never waits for the potentials. Threads past the last column compute (in-bounds) garbage that
    // the epilogue masks out, so the slot body has no per-column branches.
    const int kt = threadIdx.x;
    uint32_t slot = 0, phase = 0, qs = 0, qph = 0;
    unsigned consumed = 0, produced = 0;
    long long c_ksum = 0, c_kqw = 0;
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
    // TMEM-resident k-blocks: thread kt's words ((r * ktm + kk) * CPT + q) * 4 + v of its lane (warp w reads
    // lanes 32 (w mod 4) ..; two warps of a lane quarter split its 512 columns), loaded once per launch
    const unsigned tcols = 512u / (unsigned)((nk + 3) / 4);
    const unsigned tb = ctl[12] + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)(warp >> 2) * tcols;
    if (p.ktm > 0 && active0) {
      for (int r = 0; r < nrows; ++r)
        for (int kk = 0; kk < p.ktm; ++kk)
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            const int jv = q * nkt + kt;
            const float4 v = jv < mv ? __ldg(reinterpret_cast<const VT*>(p.C + ((size_t)(p.kres + kk) * R + i0 + r) * m) + jv)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
            asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                             tb + (unsigned)(((r * p.ktm + kk) * CPT + q) * 4)),
                         "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)), "r"(__float_as_uint(v.z)),
                         "r"(__float_as_uint(v.w)));
          }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    const int total_rows = p.iters * nrows;
    for (int rr = 0; active0 && rr < total_rows; ++rr) {
      // CTA-uniform (k-sum warps) check of the halt flag
      if (kt == 0) ctl[8] = lds_acquire(&ctl[5]);
      asm volatile("bar.sync 3, %0;" ::"r"(nkt) : "memory");
      const bool halt = ctl[8] != 0;
      asm volatile("bar.sync 3, %0;" ::"r"(nkt) : "memory");
      if (halt) break;
      const int r = rr % nrows;
      // the row's integer shifts a_ij = round(G_ij log2e/eps): s'_ij = sum_k 2^{a_ij - C_ijk log2e/eps}, one
      // rounding per term (the product is exact inside the FMA); the G-shifted S_ij of the precomputed mode is
      // rescaled by 2^{a_ij - G_ij log2e/eps} (|.| <= 1/2) to the same convention
      float gc[CPT][VEC], s[CPT][VEC], pf[CPT][VEC];
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const float gv[VEC] = {gnext[q].x, gnext[q].y, gnext[q].z, gnext[q].w};
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          gc[q][v] = (float)__float2int_rn(gv[v] * c2);
          pf[q][v] = p.pre ? ex2(fmaf(-gv[v], c2, gc[q][v])) : 1.f;
          s[q][v] = 0.f;
        }
      }
      load_g(r + 1 < nrows ? i0 + r + 1 : i0);
      const long long tk0 = p.trace ? clock64() : 0;
      int k0 = p.kres;
      if (p.kres > 0) {   // the resident k-blocks of the row, straight from shared memory (k ascending, as streamed)
        if (rr == 0) mbar_wait(resbar, 0);
        const VT* rb = reinterpret_cast<const VT*>(resid + (size_t)r * p.kres * m);
        if (!(p.diag & COT_DIAG_NO_COMPUTE)) {
          int k = 0;
          for (; k + 4 <= p.kres; k += 4) ksum4<CPT>(rb + (size_t)k * mv, mv, nkt, kt, c2, gc, s);
          for (; k < p.kres; ++k) ksum1<CPT>(rb + (size_t)k * mv, nkt, kt, c2, gc, s);
        }
      }
      if (p.ktm > 0) {   // the TMEM-resident k-blocks, four k-rows per load (the same grouping and order as ksum4)
        const unsigned tr = tb + (unsigned)(r * p.ktm * CPT * 4);
        if (!(p.diag & COT_DIAG_NO_COMPUTE))
          for (int kk = 0; kk < p.ktm; kk += 4) {
            unsigned x[16 * CPT];
#pragma unroll
            for (int h = 0; h < CPT; ++h)
              asm volatile(
                  "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                  : "=r"(x[16 * h]), "=r"(x[16 * h + 1]), "=r"(x[16 * h + 2]), "=r"(x[16 * h + 3]), "=r"(x[16 * h + 4]),
                    "=r"(x[16 * h + 5]), "=r"(x[16 * h + 6]), "=r"(x[16 * h + 7]), "=r"(x[16 * h + 8]),
                    "=r"(x[16 * h + 9]), "=r"(x[16 * h + 10]), "=r"(x[16 * h + 11]), "=r"(x[16 * h + 12]),
                    "=r"(x[16 * h + 13]), "=r"(x[16 * h + 14]), "=r"(x[16 * h + 15])
                  : "r"(tr + (unsigned)(kk * CPT * 4 + 16 * h)));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            float e[4][CPT][4];
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4)
#pragma unroll
              for (int q = 0; q < CPT; ++q)
#pragma unroll
                for (int v = 0; v < 4; ++v)
                  e[k4][q][v] = ex2(fmaf(-__uint_as_float(x[(k4 * CPT + q) * 4 + v]), c2, gc[q][v]));
#pragma unroll
            for (int q = 0; q < CPT; ++q)
#pragma unroll
              for (int v = 0; v < 4; ++v) s[q][v] += (e[0][q][v] + e[1][q][v]) + (e[2][q][v] + e[3][q][v]);
          }
        k0 = p.kres + p.ktm;
      }
      for (; k0 + KS <= n; k0 += KS) {
        mbar_wait(&full[slot], phase);
        const VT* sb = reinterpret_cast<const VT*>(ring + (size_t)slot * slot_floats);
        if (p.pre) {   // NEXT-1: the slot holds S_ij (n = KS = 1)
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            const float4 c = sb[q * nkt + kt];
            s[q][0] = c.x * pf[q][0];
            s[q][1] = c.y * pf[q][1];
            s[q][2] = c.z * pf[q][2];
            s[q][3] = c.w * pf[q][3];
          }
        } else if (!(p.diag & COT_DIAG_NO_COMPUTE)) {
          if (KS >= 4) {
#pragma unroll
            for (int q2 = 0; q2 < KS; q2 += 4) ksum4<CPT>(sb + (size_t)q2 * mv, mv, nkt, kt, c2, gc, s);
          } else {
#pragma unroll
            for (int q2 = 0; q2 < KS; ++q2) ksum1<CPT>(sb + (size_t)q2 * mv, nkt, kt, c2, gc, s);
          }
        }
        release();
      }
      if (k0 < n) {   // ragged last slot of the row (n % KS != 0)
        const int kk = n - k0;
        mbar_wait(&full[slot], phase);
        const VT* sb = reinterpret_cast<const VT*>(ring + (size_t)slot * slot_floats);
        if (!(p.diag & COT_DIAG_NO_COMPUTE)) {
          int q2 = 0;
          for (; q2 + 4 <= kk; q2 += 4) ksum4<CPT>(sb + (size_t)q2 * mv, mv, nkt, kt, c2, gc, s);
          for (; q2 < kk; ++q2) ksum1<CPT>(sb + (size_t)q2 * mv, nkt, kt, c2, gc, s);
        }
        release();
      }
      if (p.trace) c_ksum += clock64() - tk0;
      // ---- hand the row's k-sums to the epilogue warps through the queue
      const long long tqe = p.trace ? clock64() : 0;
      mbar_wait(&qempty[qs], qph ^ 1u);
      if (p.trace) c_kqw += clock64() - tqe;
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
    if (p.trace && kt == 0) {
      p.trace[bid * 16 + 3] = c_ksum;
      p.trace[bid * 16 + 9] = c_kqw;
    }
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
    if (p.ktm > 0) {   // every k-sum warp is past its last TMEM read
      asm volatile("tcgen05.fence::before_thread_sync;");
      asm volatile("bar.sync 3, %0;" ::"r"(nkt) : "memory");
      if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(ctl[12]));
    }
  } else {
    // ===================================================================== epilogue warps
    // Per iteration: (1) the row epilogues (in order): wait for the row's k-sums in the queue, then
    //   x_ij = z_hat_j - G_ij/eps, r_i = sum_j s_ij exp(x_ij - M'_i) and M_i = max_j x_ij in ONE block
    //   reduction against the previous row maximum M'_i (exact exponent split), w_hat_i, and the column
    //   partial P_j += (alpha_i/r_i) t_ij;
    // (2) the device-wide steps, with no grid barrier: the CTA's partial goes out as LL lines (each fp64 value
    //   with the iteration's generation in both 8-byte halves), the owner CTA of each column slice polls the
    //   slice's lines of every unit and sums them in unit order (deterministic), [fused multi-GPU: exchanges
    //   the slice's sums with the other ranks the same way], applies the q-update and publishes z_hat of the
    //   slice as LL lines; every CTA then polls the z lines it needs for the next iteration. The monitor is a
    //   line per CTA, summed in CTA order by every CTA (identical freeze decisions).
    const int et = threadIdx.x - nkt;
    const bool fused = p.nranks > 0;
    const bool sync = !p.rows_only && !(p.diag & COT_DIAG_NO_SYNC);
    const int ncs = fused ? p.ncs : nblk;
    const int cpc = (m + ncs - 1) / ncs;
    const int col0 = bid < ncs ? bid * cpc : m;
    const int col1 = min(m, col0 + cpc);
    const int ngrp = net >> 3;                // column pass: thread = (unit group, column of an 8-column chunk)
    const unsigned long long lep0 = sync ? *(volatile const unsigned long long*)p.lepoch : 0ull;
    const unsigned long long xep0 = fused ? *(volatile const unsigned long long*)p.xepoch : 0ull;
    uint32_t qs = 0, qph = 0;
    unsigned consumed = 0;
    int rbuf = 0;
    long long c_epi = 0, c_wait = 0, c_cmp = 0, c_red = 0, c_col = 0, c_qw = 0, c_cp1 = 0, c_pub = 0;
    bool timeout = false;
    const bool have_ref = p.state[0].iters > 0;   // w_hat holds the previous iteration's p-update
    for (int r = et; r < nrows; r += net) {
      const double a = p.alpha[p.row_begin + i0 + r];
      const double la = log(a);
      // shift reference = the row's log-sum-exp of the previous iteration, log alpha_i - w_hat_i (NaN: none)
      rowstat[r * RS + 0] = have_ref ? la - p.w_hat[p.row_begin + i0 + r] : __longlong_as_double(0x7ff8000000000000LL);
      rowstat[r * RS + 3] = la;
      rowstat[r * RS + 4] = a;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(net) : "memory");
    SolverState st = p.state[0];
    const long long iters0 = st.iters;
    double P[EPT][VEC];
    int kz[EPT][VEC];     // z_j log2e = kz_j + f_j, Fz_j = 2^{f_j} (fp64): once per column per iteration
    double Fz[EPT][VEC];
#pragma unroll
    for (int q = 0; q < EPT; ++q)
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const int jv = q * net + et;
        Fz[q][v] = split_z((jv < mv ? __ldcg(p.z_hat + VEC * jv + v) : 0.0), kz[q][v]);
        P[q][v] = 0.0;
      }
    auto need_resid = [&](int t) {
      const long long itg = iters0 + t + 1;
      return (p.tol > 0.0 && itg % p.check_every == 0) || t == p.iters - 1;
    };
    // monitor of the iteration that produced generation g: sum of the slice owners' lines in CTA order
    auto read_resid = [&](unsigned g) {
      const uint4* rl = p.rlines + (size_t)(g & 1u) * p.lcap;
      double v = 0.0;
      for (int b = et; b < ncs; b += net) {
        double x;
        timeout |= !poll_line(rl + b, g, x);
        v += x;
      }
      return cblk_sum1(v, red2, rbuf, net, nk);
    };
    // log beta_j of the first 8 columns of this CTA's slice (the usual whole slice), once per launch
    const bool own0 = sync && et < 8 && col0 + et < col1;   // rows_only launches have no beta
    const double beta0 = own0 ? p.beta[col0 + et] : 1.0;
    const double lbeta0 = own0 ? log(beta0) : 0.0;
    double zown0 = own0 ? __ldcg(p.z_hat + col0 + et) : 0.0;   // this thread's z_hat of the slice, kept in a register
    int done = 0;   // iterations completed (q-update applied) in this launch
    bool halted = false;
    // ---- w_hat of this CTA's rows, LSE_i = shift_i + log r_i, from the row statistics of the last completed
    // iteration: written once per launch (after the last iteration, or where the launch halts), not per iteration;
    // log without MUFU (the k-sum warps keep it busy)
    auto write_w_hat = [&]() {
      if (et < 32) {   // the writer's warp (__syncwarp orders its shared-memory writes for the lanes)
        __syncwarp();
        for (int r = et; r < nrows; r += 32)
          p.w_hat[p.row_begin + i0 + r] = rowstat[r * RS + 3] - (rowstat[r * RS + 1] + log_nomufu(rowstat[r * RS + 2]));
      }
    };
    for (int t = 0; active0 && t < p.iters; ++t) {
      if (t > 0 && sync) {
        // ---- z_hat of generation g (the q-update of iteration t-1) and, if due, its monitor
        const long long tw0 = p.trace ? clock64() : 0;
        const unsigned g = (unsigned)(lep0 + t);
#pragma unroll
        for (int q = 0; q < EPT; ++q) {
          const int jv = q * net + et;
          if (jv < mv) {   // the 4 lines of this thread's columns, re-polled together while any is missing
            uint4 zl[VEC];
            unsigned todo = (1u << VEC) - 1u;
            const unsigned long long tz0 = gtimer();
            while (todo) {
#pragma unroll
              for (int v = 0; v < VEC; ++v)
                if (todo & (1u << v)) {
                  zl[v] = ld_line(p.zlines + VEC * jv + v);
                  if (ll_ready(zl[v], g)) todo &= ~(1u << v);
                }
              if (todo && gtimer() - tz0 > kPeerTimeoutNs) {
                timeout = true;
                break;
              }
            }
#pragma unroll
            for (int v = 0; v < VEC; ++v) Fz[q][v] = split_z(ll_value(zl[v]), kz[q][v]);
          }
        }
        if (need_resid(t - 1)) st.residual = read_resid(g) * (double)n;
        if (p.trace) c_wait += clock64() - tw0;
        // a CTA that gave up waiting halts (its peers then time out on its lines and halt too); no global read
        // of the state flags on the per-iteration critical path. `timeout` is per thread (only the threads whose
        // lines went missing see it): OR it over the epilogue warps first, so the whole CTA takes the same exit
        // (the named barriers and the queue's mbarrier phases stay matched).
        timeout = bar_red_or(timeout, net);
        if (timeout) halted = true;
        if (p.tol > 0.0 && st.iters % p.check_every == 0 && st.residual <= p.tol) {
          st.active = 0;
          st.converged = 1;
          halted = true;
        }
        if (halted) {
          st.active = 0;
          if (et == 0) sts_release(&ctl[5], 1u);   // stop the k-sum warps (their rows are drained below)
          write_w_hat();                            // the row statistics of iteration t - 1 are still in place
          break;
        }
      }
      if (p.rpw) {
        // ---- row-per-warp epilogue (rows per CTA <= 8): warp w takes rows w, w + ne, ...; per row the terms
        // t_ij = s'_ij 2^{kz_j - kM_i - a_ij} Fz_j are summed by warp shuffles and stored (fp64) in the row's
        // slot of a shared-memory tile; after one epilogue barrier every thread forms its columns' partial
        // P_j = sum_i (alpha_i / r_i) t_ij over the rows in row order. kM_i: the previous iteration's shift +
        // floor(log2 r_i); a row whose sum leaves [1e-280, 1e280] (first iteration, or a jump of the
        // potentials) is redone with the exact kM_i = max_j (kz_j - a_ij) (warp-local, one REDUX).
        const long long te0 = p.trace ? clock64() : 0;
#pragma unroll
        for (int q = 0; q < EPT; ++q) {
          const int jv = q * net + et;
          if (jv < mv) {
            reinterpret_cast<int4*>(zks)[jv] = make_int4(kz[q][0], kz[q][1], kz[q][2], kz[q][3]);
            reinterpret_cast<double2*>(zfs)[2 * jv] = make_double2(Fz[q][0], Fz[q][1]);
            reinterpret_cast<double2*>(zfs)[2 * jv + 1] = make_double2(Fz[q][2], Fz[q][3]);
          }
        }
        cbar(net);
        const int ew = et >> 5;
        const int nq = (mv + 31) >> 5;
        const int4* zk4 = reinterpret_cast<const int4*>(zks);
        const double2* zf2 = reinterpret_cast<const double2*>(zfs);
        for (int r = ew; r < nrows; r += ne) {
          const unsigned g = (unsigned)t * (unsigned)nrows + (unsigned)r;   // FIFO position of the row
          const uint32_t slot = g % (unsigned)QN, ph = (g / (unsigned)QN) & 1u;
          mbar_wait(&qfull[slot], ph);
          const float4* srow = reinterpret_cast<const float4*>(queue + (size_t)slot * m);
          const int4* arow = reinterpret_cast<const int4*>(gsh + (size_t)r * m);
          double2* trow = reinterpret_cast<double2*>(wpart + (size_t)r * m);
          auto row_terms = [&](int kM) {
            double lsum = 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {   // nq <= 8 (m <= 1024): unrolled, predicated
              const int jv = q * 32 + lane;
              if (q < nq && jv < mv) {
                const float4 s4 = srow[jv];
                const int4 a4 = arow[jv], k4 = zk4[jv];
                const double2 fa = zf2[2 * jv], fb = zf2[2 * jv + 1];
                const double t0 = ldexp_pos(s4.x, k4.x - a4.x - kM) * fa.x;
                const double t1 = ldexp_pos(s4.y, k4.y - a4.y - kM) * fa.y;
                const double t2 = ldexp_pos(s4.z, k4.z - a4.z - kM) * fb.x;
                const double t3 = ldexp_pos(s4.w, k4.w - a4.w - kM) * fb.y;
                trow[2 * jv] = make_double2(t0, t1);
                trow[2 * jv + 1] = make_double2(t2, t3);
                lsum += (t0 + t1) + (t2 + t3);
              }
            }
            return warp_sum(lsum);
          };
          // deterministic mode: always the exact shift (a function of z and the row only, so iterates do not
          // depend on launch boundaries either)
          const double ref = p.det ? __longlong_as_double(0x7ff8000000000000LL) : rowstat[r * RS + 0];
          int kM = ref == ref ? __double2int_rn(ref * COT_LOG2E) : 0;
          double rsum = ref == ref ? row_terms(kM) : 0.0;
          if (!(rsum >= 1e-280 && rsum <= 1e280)) {   // warp-uniform: exact shift, terms again
            int emax = -0x7fffffff;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int jv = q * 32 + lane;
              if (q < nq && jv < mv) {
                const int4 a4 = arow[jv], k4 = zk4[jv];
                emax = max(emax, max(max(k4.x - a4.x, k4.y - a4.y), max(k4.z - a4.z, k4.w - a4.w)));
              }
            }
            kM = __reduce_max_sync(0xffffffffu, emax);
            rsum = row_terms(kM);
          }
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&qempty[slot]);
            rowstat[r * RS + 0] = (double)(kM + ((__double2hiint(rsum) >> 20) - 1023)) * COT_LN2;   // next shift
            rowstat[r * RS + 1] = (double)kM * COT_LN2;   // shift used for r_i (natural units)
            rowstat[r * RS + 2] = rsum;
            rowstat[r * RS + 5] = rowstat[r * RS + 4] * rcp_nomufu(rsum);   // alpha_i / r_i
          }
        }
        // the FIFO position after this iteration's rows (the drain after a halt continues from here)
        consumed += (unsigned)nrows;
        qs = consumed % (unsigned)QN;
        qph = (consumed / (unsigned)QN) & 1u;
        cbar(net);   // every row's terms and statistics are in shared memory
        double rho8[8];   // (deterministic mode: the fixed-point partial is formed when the lines are written)
#pragma unroll
        for (int r = 0; r < 8; ++r) rho8[r] = r < nrows ? rowstat[r * RS + 5] : 0.0;
#pragma unroll
        for (int q = 0; q < EPT; ++q) {
          const int jv = q * net + et;
          if (jv < mv && !p.det) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
              double acc = 0.0;   // rows in order
#pragma unroll
              for (int r = 0; r < 8; ++r)
                if (r < nrows) acc = fma(rho8[r], wpart[(size_t)r * m + VEC * jv + v], acc);
              P[q][v] = acc;
            }
          }
        }
        if (p.trace) c_epi += clock64() - te0;
      } else {
      // rows in batches of RB: one block reduction (the RB row sums) per batch; the batch's k-sums are read
        // straight from the queue slots (released after the batch) and -G/eps from shared memory
        for (int r0 = 0; r0 < nrows; r0 += RB) {
          const int nb = min(RB, nrows - r0);
          uint32_t qsb[RB];
          {
            uint32_t q2 = qs, ph2 = qph;
            const long long tq0 = p.trace ? clock64() : 0;
  #pragma unroll
            for (int b = 0; b < RB; ++b) {
              qsb[b] = q2;
              if (b < nb) {
                mbar_wait(&qfull[q2], ph2);
                if (++q2 == (uint32_t)QN) {
                  q2 = 0;
                  ph2 ^= 1u;
                }
              }
            }
            if (p.trace) c_qw += clock64() - tq0;
          }
          const long long te0 = p.trace ? clock64() : 0;
  #pragma unroll
          for (int b = 1; b < RB; ++b)
            if (b >= nb) qsb[b] = qsb[0];          // branch-free: unused rows read a valid slot, masked below
          // ---- the row epilogues: t_ij = s_ij exp(x_ij - Mref_i), x_ij = z_j - G_ij/eps, with Mref_i the row's
          // log-sum-exp of the previous iteration (so x - Mref <= ~log(n m) unless z jumped); r_i = sum_j t_ij
          // in one block reduction for the batch. A batch with a row sum outside [1e-280, 1e280] (no reference
          // yet, or a jump of the potentials) is redone in the exact two-pass form (maximum first).
          double Mref[RB], sm[RB], tt[RB][EPT][VEC];
  #pragma unroll
          for (int b = 0; b < RB; ++b) {
            Mref[b] = rowstat[(r0 + (b < nb ? b : 0)) * RS + 0];
            sm[b] = 0.0;
          }
          const bool stale = Mref[0] == Mref[0];      // the CTA's rows get their references together
          auto batch_terms = [&](bool use) {
  #pragma unroll
            for (int b = 0; b < RB; ++b) {
              if (b >= nb) {   // CTA-uniform: short batches (e.g. one row per CTA) skip the unused rows
  #pragma unroll
                for (int q = 0; q < EPT; ++q)
  #pragma unroll
                  for (int v = 0; v < VEC; ++v) tt[b][q][v] = 0.0;
                continue;
              }
              const int rb = r0 + (b < nb ? b : 0);
              const int kM = __double2int_rn(Mref[b] * COT_LOG2E);   // integer row shift (exact: no rounded factor)
  #pragma unroll
              for (int q = 0; q < EPT; ++q) {
                const int jv = q * net + et;
                const bool ok = use && jv < mv && b < nb;
                const int jc = jv < mv ? jv : 0;
                const float4 s4 = reinterpret_cast<const VT*>(queue + (size_t)qsb[b] * m)[jc];
                const int4 a4 = reinterpret_cast<const int4*>(gsh + (size_t)rb * m)[jc];
                const double t0 = ldexp_pos(s4.x, kz[q][0] - kM - a4.x) * Fz[q][0];
                const double t1 = ldexp_pos(s4.y, kz[q][1] - kM - a4.y) * Fz[q][1];
                const double t2 = ldexp_pos(s4.z, kz[q][2] - kM - a4.z) * Fz[q][2];
                const double t3 = ldexp_pos(s4.w, kz[q][3] - kM - a4.w) * Fz[q][3];
                tt[b][q][0] = ok ? t0 : 0.0;
                tt[b][q][1] = ok ? t1 : 0.0;
                tt[b][q][2] = ok ? t2 : 0.0;
                tt[b][q][3] = ok ? t3 : 0.0;
                sm[b] += (tt[b][q][0] + tt[b][q][1]) + (tt[b][q][2] + tt[b][q][3]);
              }
            }
          };
          batch_terms(stale);
          const long long te1 = p.trace ? clock64() : 0;
          cblk_sumN<RB>(sm, red2, rbuf, net, nk);
          if (p.trace) {
            c_cmp += te1 - te0;
            c_red += clock64() - te1;
          }
          bool redo = false;
  #pragma unroll
          for (int b = 0; b < RB; ++b) redo |= b < nb && !(sm[b] >= 1e-280 && sm[b] <= 1e280);
          if (redo) {   // block-uniform (sm is the block total): exact two-pass for the whole batch
            double mx[RB];
  #pragma unroll
            for (int b = 0; b < RB; ++b) {
              mx[b] = -INFINITY;
              const int rb = r0 + (b < nb ? b : 0);
  #pragma unroll
              for (int q = 0; q < EPT; ++q)
  #pragma unroll
                for (int v = 0; v < VEC; ++v) {
                  const int jv = q * net + et;
                  if (jv < mv && b < nb)   // the largest kz_j - a_ij: every term <= 2^{1/2} s'_ij, the largest >= 1/2
                    mx[b] = fmax(mx[b], (double)(kz[q][v] - gsh[(size_t)rb * m + VEC * jv + v]));
                }
            }
            cblk_maxN<RB>(mx, red2, rbuf, net, nk);
  #pragma unroll
            for (int b = 0; b < RB; ++b) {
              Mref[b] = b < nb ? mx[b] * COT_LN2 : 0.0;
              sm[b] = 0.0;
            }
            batch_terms(true);
            cblk_sumN<RB>(sm, red2, rbuf, net, nk);
          }
          // release the batch's queue slots
          __syncwarp();
  #pragma unroll
          for (int b = 0; b < RB; ++b) {
            if (b >= nb) break;
            if (lane == 0) mbar_arrive(&qempty[qs]);
            ++consumed;
            if (++qs == (uint32_t)QN) {
              qs = 0;
              qph ^= 1u;
            }
          }
  #pragma unroll
          for (int b = 0; b < RB; ++b) {
            if (b >= nb) break;
            const int r = r0 + b;
            const double rsum = sm[b];
            const double rinv = rcp_nomufu(rsum);   // alpha_i / r_i
            const double rho = rowstat[r * RS + 4] * rinv;
            if (et == 0) {   // the shift used for r_i, r_i, and the next iteration's shift: kM + floor(log2 r_i)
              const int kM = __double2int_rn(Mref[b] * COT_LOG2E);
              rowstat[r * RS + 0] = (double)(kM + ((__double2hiint(rsum) >> 20) - 1023)) * COT_LN2;
              rowstat[r * RS + 1] = (double)kM * COT_LN2;
              rowstat[r * RS + 2] = rsum;
            }
  #pragma unroll
            for (int q = 0; q < EPT; ++q)
  #pragma unroll
              for (int v = 0; v < VEC; ++v) P[q][v] = fma(rho, tt[b][q][v], P[q][v]);
          }
          if (p.trace) c_epi += clock64() - te0;
        }
      }
      if (p.rows_only) {   // cerot_rows: the plain fp64 partial, no device-wide step
        write_w_hat();
#pragma unroll
        for (int q = 0; q < EPT; ++q) {
          const int jv = q * net + et;
          if (jv < mv)
            reinterpret_cast<double4*>(p.partials + (size_t)u * m)[jv] = make_double4(P[q][0], P[q][1], P[q][2], P[q][3]);
        }
        done = 1;
        break;
      }
      if (!sync) {   // diagnostics (COT_DIAG_NO_SYNC): no column pass, z_hat unchanged
        write_w_hat();
#pragma unroll
        for (int q = 0; q < EPT; ++q)
#pragma unroll
          for (int v = 0; v < VEC; ++v) P[q][v] = 0.0;
        st.iters += 1;
        ++done;
        continue;
      }
      const long long tp0 = p.trace ? clock64() : 0;
      // ---- publish the column partial of iteration t as LL lines of generation g1
      const unsigned g1 = (unsigned)(lep0 + t + 1);
      if (p.det) {   // 128-bit fixed point: lines 2j (low word) and 2j + 1 (high word) of a 2m-line unit row
        uint4* pl = p.plines + ((size_t)(g1 & 1u) * p.lcap + u) * (2 * m);
#pragma unroll
        for (int q = 0; q < EPT; ++q) {
          const int jv = q * net + et;
          if (jv < mv) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
              const int j = VEC * jv + v;
              unsigned long long lo = 0, hi = 0;
              for (int r = 0; r < nrows; ++r) fx_acc(rowstat[r * RS + 5] * wpart[(size_t)r * m + j], lo, hi);
              st_line(pl + 2 * j, ll_pack(bitsd(lo), g1));
              st_line(pl + 2 * j + 1, ll_pack(bitsd(hi), g1));
            }
          }
        }
      } else {
        uint4* pl = p.plines + ((size_t)(g1 & 1u) * p.lcap + u) * m;
#pragma unroll
        for (int q = 0; q < EPT; ++q) {
          const int jv = q * net + et;
          if (jv < mv) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) st_line(pl + VEC * jv + v, ll_pack(P[q][v], g1));
          }
#pragma unroll
          for (int v = 0; v < VEC; ++v) P[q][v] = 0.0;
        }
      }
      if (t == p.iters - 1) write_w_hat();
      // ---- column pass of this CTA's slice: c_j = sum_u P_uj in unit order; q-update; z lines
      const long long tc0 = p.trace ? clock64() : 0;
      if (p.trace) c_pub += tc0 - tp0;
      double dev = 0.0;
      const uint4* plr = p.plines + (size_t)(g1 & 1u) * p.lcap * m;
      if (p.det) {
        // ---- deterministic column pass: the units' 128-bit partials summed exactly (any order), the rank sums
        // likewise; one conversion to fp64 per column, identical for every row partition
        const uint4* pld = p.plines + (size_t)(g1 & 1u) * p.lcap * (2 * m);
        for (int cb = col0; cb < col1; cb += 8) {
          const int c = et & 7, grp = et >> 3;
          const bool colok = cb + c < col1;
          unsigned long long alo = 0, ahi = 0;
          for (int ub = grp; ub < nblk; ub += 4 * ngrp) {   // 4 units (8 lines) in flight per thread
            uint4 l[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int u2 = ub + (k >> 1) * ngrp;
              l[k] = (colok && u2 < nblk) ? ld_line(pld + (size_t)u2 * (2 * m) + 2 * (cb + c) + (k & 1))
                                          : make_uint4(0u, g1, 0u, g1);
            }
            unsigned todo = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (colok && ub + (k >> 1) * ngrp < nblk && !ll_ready(l[k], g1)) todo |= 1u << k;
            const unsigned long long tp0 = todo ? gtimer() : 0ull;
            while (todo) {
#pragma unroll
              for (int k = 0; k < 8; ++k)
                if (todo & (1u << k)) {
                  l[k] = ld_line(pld + (size_t)(ub + (k >> 1) * ngrp) * (2 * m) + 2 * (cb + c) + (k & 1));
                  if (ll_ready(l[k], g1)) todo &= ~(1u << k);
                }
              if (todo && gtimer() - tp0 > kPeerTimeoutNs) {
                timeout = true;
                break;
              }
            }
#pragma unroll
            for (int k = 0; k < 8; k += 2) fx_add(alo, ahi, dbits(ll_value(l[k])), dbits(ll_value(l[k + 1])));
          }
          if (p.trace) c_cp1 += clock64() - tc0;
#pragma unroll
          for (int o = 8; o <= 16; o <<= 1) {
            const unsigned long long olo = __shfl_xor_sync(0xffffffffu, alo, o);
            const unsigned long long ohi = __shfl_xor_sync(0xffffffffu, ahi, o);
            fx_add(alo, ahi, olo, ohi);
          }
          asm volatile("bar.sync 1, %0;" ::"r"(net) : "memory");
          if (lane < 8) {
            xs[(grp >> 2) * 8 + c] = bitsd(alo);
            xs[64 + (grp >> 2) * 8 + c] = bitsd(ahi);
          }
          asm volatile("bar.sync 1, %0;" ::"r"(net) : "memory");
          double cj = 0.0;
          unsigned long long slo = 0, shi = 0;
          if (et < 8)
            for (int w2 = 0; w2 < (ngrp >> 2); ++w2) fx_add(slo, shi, dbits(xs[w2 * 8 + et]), dbits(xs[64 + w2 * 8 + et]));
          if (fused) {   // the slice's 128-bit sums to every rank (2 lines each), then all ranks' sums, exactly
            const int nr = p.nranks;
            const unsigned xg = (unsigned)(xep0 + t + 1);
            const int par = (int)(xg & 1u);
            if (et < 8 && cb + et < col1) {
              const uint4 llo = ll_pack(bitsd(slo), xg), lhi = ll_pack(bitsd(shi), xg);
              for (int q = 0; q < nr; ++q) {
                uint4* dst = p.xpeer[q] + ((size_t)(par * nr + p.rank)) * (2 * m) + 2 * (cb + et);
                st_line(dst, llo);
                st_line(dst + 1, lhi);
              }
            }
            for (int q = et >> 3; q < nr && colok; q += ngrp) {
              double vlo, vhi;
              const uint4* src = p.xpeer[p.rank] + ((size_t)(par * nr + q)) * (2 * m) + 2 * (cb + c);
              timeout |= !poll_line(src, xg, vlo);
              timeout |= !poll_line(src + 1, xg, vhi);
              xs[kRankScratch + q * 8 + c] = vlo;
              xs[kRankScratch + kMaxRanks * 8 + q * 8 + c] = vhi;
            }
            asm volatile("bar.sync 1, %0;" ::"r"(net) : "memory");
            if (et < 8) {
              slo = shi = 0;
              for (int q2 = 0; q2 < nr; ++q2)
                fx_add(slo, shi, dbits(xs[kRankScratch + q2 * 8 + et]), dbits(xs[kRankScratch + kMaxRanks * 8 + q2 * 8 + et]));
            }
          }
          if (et < 8 && cb + et < col1) {
            cj = fx_to_double(slo, shi);
            const int j = cb + et;
            const double bj = cb == col0 ? beta0 : p.beta[j];
            dev += fabs(cj - bj);
            if (!(cj >= 1e-28)) atomicOr(&p.state[0].flags, (int)STATE_UNDERFLOW);
            const double zold = cb == col0 ? zown0 : __ldcg(p.z_hat + j);
            const double zj = zold + ((cb == col0 ? lbeta0 : log(bj)) - log_nomufu(cj));
            if (cb == col0) zown0 = zj;
            p.z_hat[j] = zj;
            st_line(p.zlines + j, ll_pack(zj, g1));
          }
        }
      } else
      for (int cb = col0; cb < col1; cb += 8) {
        const int c = et & 7, grp = et >> 3;
        const bool colok = cb + c < col1;
        double acc = 0.0;
        for (int ub = grp; ub < nblk; ub += 8 * ngrp) {   // 8 lines in flight per thread, unit order kept
          uint4 l[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int u2 = ub + k * ngrp;
            l[k] = (colok && u2 < nblk) ? ld_line(plr + (size_t)u2 * m + cb + c) : make_uint4(0u, g1, 0u, g1);
          }
          // re-poll every line still missing in the same round (one round trip per round, not per line)
          unsigned todo = 0;
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (colok && ub + k * ngrp < nblk && !ll_ready(l[k], g1)) todo |= 1u << k;
          const unsigned long long tp0 = todo ? gtimer() : 0ull;
          while (todo) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (todo & (1u << k)) {
                l[k] = ld_line(plr + (size_t)(ub + k * ngrp) * m + cb + c);
                if (ll_ready(l[k], g1)) todo &= ~(1u << k);
              }
            if (todo && gtimer() - tp0 > kPeerTimeoutNs) {
              timeout = true;
              break;
            }
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) acc += ll_value(l[k]);   // unit order
        }
        if (p.trace) c_cp1 += clock64() - tc0;
        // groups of a warp (lanes c, c+8, c+16, c+24) by two shuffle levels, then the warps in order
        acc += __shfl_xor_sync(0xffffffffu, acc, 8);
        acc += __shfl_xor_sync(0xffffffffu, acc, 16);
        asm volatile("bar.sync 1, %0;" ::"r"(net) : "memory");   // previous chunk's readers of xs are done
        if (lane < 8) xs[(grp >> 2) * 8 + c] = acc;
        asm volatile("bar.sync 1, %0;" ::"r"(net) : "memory");
        double cj = 0.0;
        if (et < 8) {
          double v8[8];
#pragma unroll
          for (int w2 = 0; w2 < 8; ++w2) v8[w2] = w2 < (ngrp >> 2) ? xs[w2 * 8 + et] : 0.0;
#pragma unroll
          for (int h = 4; h >= 1; h >>= 1)
#pragma unroll
            for (int w2 = 0; w2 < h; ++w2) v8[w2] += v8[w2 + h];
          cj = v8[0];
        }
        if (fused) {
          // ---- the exchange step across GPUs: this rank's slice sums -> every rank's x-lines (NVLink peer
          // stores), then all ranks' lines of the slice from this rank's buffer, summed in rank order
          const int nr = p.nranks;
          const unsigned xg = (unsigned)(xep0 + t + 1);
          const int par = (int)(xg & 1u);
          if (et < 8 && cb + et < col1) {
            const uint4 line = ll_pack(cj, xg);
            for (int q = 0; q < nr; ++q) st_line(p.xpeer[q] + ((size_t)(par * nr + p.rank)) * m + cb + et, line);
          }
          for (int q = et >> 3; q < nr && colok; q += ngrp) {
            double v;
            timeout |= !poll_line(p.xpeer[p.rank] + ((size_t)(par * nr + q)) * m + cb + c, xg, v);
            xs[kRankScratch + q * 8 + c] = v;
          }
          asm volatile("bar.sync 1, %0;" ::"r"(net) : "memory");
          if (et < 8) {
            cj = 0.0;
            for (int q2 = 0; q2 < nr; ++q2) cj += xs[kRankScratch + q2 * 8 + et];
          }
        }
        if (et < 8 && cb + et < col1) {
          const int j = cb + et;
          const double bj = cb == col0 ? beta0 : p.beta[j];
          dev += fabs(cj - bj);
          if (!(cj >= 1e-28)) atomicOr(&p.state[0].flags, (int)STATE_UNDERFLOW);
          const double zold = cb == col0 ? zown0 : __ldcg(p.z_hat + j);
          const double zj = zold + ((cb == col0 ? lbeta0 : log(bj)) - log_nomufu(cj));
          if (cb == col0) zown0 = zj;
          p.z_hat[j] = zj;
          st_line(p.zlines + j, ll_pack(zj, g1));
        }
      }
      if (timeout) atomicOr(&p.state[0].flags, (int)STATE_PEER_TIMEOUT);
      if (p.trace) c_col += clock64() - tc0;
      if (need_resid(t)) {
        dev = cblk_sum1(dev, red2, rbuf, net, nk);
        if (et == 0 && bid < ncs) st_line(p.rlines + (size_t)(g1 & 1u) * p.lcap + bid, ll_pack(dev, g1));
      }
      st.iters += 1;
      ++done;
    }
    if (sync && active0 && !halted && done > 0) {   // monitor + freeze rule of the last iteration
      const unsigned g = (unsigned)(lep0 + done);
      st.residual = read_resid(g) * (double)n;
      if (p.tol > 0.0 && st.iters % p.check_every == 0 && st.residual <= p.tol) {
        st.active = 0;
        st.converged = 1;
      }
    }
    if (bid == 0 && et == 0 && active0 && !p.rows_only) {
      SolverState out = p.state[0];
      out.iters = st.iters;
      out.residual = st.residual;
      out.active = st.active;
      out.converged = st.converged;
      p.state[0] = out;
      if (sync) *(volatile unsigned long long*)p.lepoch = lep0 + (unsigned long long)done;
      if (fused) *(volatile unsigned long long*)p.xepoch = xep0 + (unsigned long long)done;
    }
    if (timeout) atomicOr(&p.state[0].flags, (int)STATE_PEER_TIMEOUT);
    if (p.trace && et == net - 32) {   // the last epilogue warp's view (skew diagnostics)
      p.trace[bid * 16 + 12] = c_cmp;
      p.trace[bid * 16 + 13] = c_red;
      p.trace[bid * 16 + 14] = c_epi;
      p.trace[bid * 16 + 15] = c_wait;
    }
    if (p.trace && et == 0) {
      p.trace[bid * 16 + 4] = c_epi;
      p.trace[bid * 16 + 5] = c_wait;
      p.trace[bid * 16 + 2] = c_cmp;
      p.trace[bid * 16 + 6] = c_red;
      p.trace[bid * 16 + 7] = c_col;
      p.trace[bid * 16 + 8] = c_qw;
      p.trace[bid * 16 + 10] = c_cp1;
      p.trace[bid * 16 + 11] = c_pub;
    }
    // ---- drain the queue after a halt: consume every row the k-sum warps still produce (row-per-warp mode:
    // one warp, the slots count one arrival)
    while (!p.rpw || et < 32) {
      const unsigned kdone = lds_volatile(&ctl[7]);
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
      } else if (kdone) {
        if (consumed >= lds_volatile(&ctl[6])) break;
      }
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------------------------------------ kernels
template <int CPT, int EPT, int KS>
__global__ void __launch_bounds__(416, 1) k_iter_tma(const __grid_constant__ TmaParams p) {
  iter_tma_body<CPT, EPT, KS>(p, blockIdx.x, gridDim.x);
}

// Emulated multi-rank launch (one GPU): virtual rank v runs on CTAs [base[v], base[v+1]) with its own
// shard, workspace and exchange lines -- the same body and the same exchange protocol as the per-GPU
// launch, in ONE cooperative grid so that the ranks' spins on each other's lines are co-resident.
struct TmaMulti {
  TmaParams rp[kMaxRanks];
  int base[kMaxRanks + 1];
  int nv;
};
template <int CPT, int EPT, int KS>
__global__ void __launch_bounds__(416, 1) k_iter_tma_emu(const __grid_constant__ TmaMulti pm) {
  int v = 0;
  while (v + 1 < pm.nv && (int)blockIdx.x >= pm.base[v + 1]) ++v;
  iter_tma_body<CPT, EPT, KS>(pm.rp[v], (int)blockIdx.x - pm.base[v], pm.base[v + 1] - pm.base[v]);
}

// ------------------------------------------------------------------------------------------ launcher
bool tma_eligible(const IterArgs& a, int sms) {
  if (sms <= 0) sms = device_sm_count();
  const int64_t rpu = unit_plan(1, a.R, sms).rpu;   // the shifts a_ij of a CTA's rows (int32) fit in <= 64 KB
  return a.dtype == COT_F32 && a.B == 1 && a.m % 4 == 0 && a.m <= 1024 && rpu * a.m * 4 <= 65536 &&
         !(a.flags & COT_FORCE_LDG);
}

namespace {
struct TmaCfg {
  int cpt, ept, KS, threads, grid;
  size_t smem;
  void* fn;       // k_iter_tma instance
  void* fn_emu;   // k_iter_tma_emu instance
};

// Parameters + launch configuration of the persistent kernel for one (shard of a) problem on `sms` SMs.
cudaError_t tma_config(const IterArgs& a, const Workspace& ws, int iters, bool rows_only, int parity, int sms,
                       TmaParams* pp, TmaCfg* cfg) {
  TmaParams& p = *pp;
  memset(&p, 0, sizeof(p));
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
  // Warp roles (13 warps at m = 1024, 128 registers): a long k-sum per row (n >= 16: the HBM-bound stream)
  // gets 8 k-sum warps and 4 epilogue warps (2 float4 each); a short one (latency-bound: the epilogue and
  // the device-wide steps dominate) gets 4 k-sum warps (2 float4 each) and 8 epilogue warps.
  const bool long_ksum =
      getenv("COT_LONG_KSUM") ? atoi(getenv("COT_LONG_KSUM")) != 0 : a.n * unit_plan(1, a.R, sms).rpu >= 128;
  const int kmax = long_ksum ? 8 : 4;
  int cpt = 1;
  while ((mv + 32 * cpt - 1) / (32 * cpt) > kmax) cpt *= 2;
  p.nk = (mv + 32 * cpt - 1) / (32 * cpt);
  p.ne = std::max(1, std::min(long_ksum ? 4 : 8, (mv + 31) / 32));
  if (const char* ev = getenv("COT_NE")) p.ne = std::max(1, std::min(8, atoi(ev)));   // tuning experiments
  int ept = 1;
  while ((mv + 32 * p.ne - 1) / (32 * p.ne) > ept) ept *= 2;
  if (cpt > 2 || ept > 2 || (cpt == 2 && ept == 2)) return cudaErrorInvalidValue;
  // ---- TMA ring and row queue
  const int row_bytes = m * 4;
  int KS = 1;
  int ks_bytes = 32768;   // 32 KB slots: >= 4 in flight per SM at m = 1024 (measured best on C4)
  if (const char* ev = getenv("COT_SLOT_BYTES")) ks_bytes = atoi(ev);   // tuning experiments
  while (KS * 2 <= 16 && KS * 2 * row_bytes <= ks_bytes && KS * 2 <= (int)a.n) KS *= 2;
  p.KS = KS;
  const size_t slot_bytes = (size_t)p.KS * row_bytes;
  // row-queue depth: 6 (the smem it frees goes to the TMA ring: C4, 7 rows per CTA, 32.0 -> 31.0 us per
  // iteration with the TMEM / L2-resident blocks; 4-6 measured flat)
  p.qn = std::max(1, std::min(p.rpu, 6));
  if (const char* ev = getenv("COT_QN")) p.qn = std::max(1, atoi(ev));
  p.qn = std::max(p.qn, std::min(p.rpu, 4));   // the epilogue holds up to one batch (<= 4 rows) of queue slots
  const size_t gsh_bytes = (size_t)p.rpu * m * 4;   // the integer shifts a_ij
  p.gsh = 1;
  if (gsh_bytes > 64 * 1024) return cudaErrorInvalidConfiguration;   // see tma_eligible
  // row-per-warp epilogue for CTAs with <= 8 rows and one float4 of columns per epilogue thread (C3: 7 rows,
  // 10.5 -> 9.0 us/iteration; the 8-way C4 shard: 1 row, 8.3 -> 8.0 us); COT_RPW=0 disables (comparison)
  const char* rpwv = getenv("COT_RPW");
  p.det = (a.flags & COT_DETERMINISTIC) ? 1 : 0;
  if (p.det && (p.rpu > 8 || rows_only)) return cudaErrorInvalidValue;   // the deterministic mode needs rpw
  p.rpw = ((ept == 1 && p.rpu <= 8 && !(rpwv && atoi(rpwv) == 0)) || p.det) ? 1 : 0;
  // the row-per-warp epilogue waits for all rows of an iteration before it releases their slots: the queue must
  // hold every row of the unit
  if (p.rpw) p.qn = std::max(p.qn, p.rpu);
  const size_t rpw_bytes = p.rpw ? (size_t)m * 12 + (size_t)p.rpu * m * 8 : 0;
  const size_t queue_bytes = (size_t)p.qn * row_bytes + (p.gsh ? gsh_bytes : 0) + (size_t)p.rpu * 6 * 8 +
                             (size_t)kColScratch * 8 + rpw_bytes;
  const size_t budget = 220 * 1024;
  if (queue_bytes + 2 * slot_bytes + 4096 > budget) return cudaErrorInvalidConfiguration;
  // Resident k-blocks: shared memory the ring does not need (beyond kMinSlots slots in flight) holds the first
  // kres k-blocks of every row of the unit for the whole launch, so only n - kres blocks per row are re-streamed
  // each iteration (every Gibbs term is still evaluated every iteration; the bytes come from on-chip memory).
  // Not for single-iteration launches (nothing to reuse) or the precomputed mode. COT_KRES overrides.
  int kMinSlots = 4;
  if (const char* ev = getenv("COT_MIN_SLOTS")) kMinSlots = std::max(2, atoi(ev));   // tuning experiments
  p.kres = 0;
  if (!rows_only && iters > 1 && !(a.flags & COT_PRECOMPUTED)) {
    const size_t fixed = queue_bytes + 4096 + (size_t)kMinSlots * slot_bytes;
    const size_t per_k = (size_t)p.rpu * row_bytes;
    if (budget > fixed) p.kres = (int)std::min<size_t>((size_t)a.n, (budget - fixed) / per_k);
  }
  if (const char* ev = getenv("COT_KRES")) {
    const int want = atoi(ev);
    if (want >= 0) p.kres = std::min(p.kres, want);
  }
  // a multiple of 4: the k-sum's blocks of four k-rows then start at the same k whether a block is resident or
  // streamed, so the sums (and every iterate) do not depend on kres -- a single-iteration launch (kres = 0)
  // continues a resident launch bit for bit
  if (p.kres < (int)a.n) p.kres &= ~3;
  const size_t resid_bytes = (size_t)p.rpu * p.kres * row_bytes;
  // TMEM-resident k-blocks (after the shared-memory ones): each k-sum thread holds 4 * CPT words per (row, k-block)
  // of its 512 / ceil(nk / 4) TMEM columns; a multiple of 4 k-blocks (the k-sum grouping); COT_KTM overrides
  p.ktm = 0;
  if (!rows_only && iters > 1 && !(a.flags & COT_PRECOMPUTED) && p.kres < (int)a.n) {
    const int words = 512 / ((p.nk + 3) / 4);
    p.ktm = std::min((int)a.n - p.kres, words / (p.rpu * cpt * 4)) & ~3;
    if (const char* ev = getenv("COT_KTM")) p.ktm = std::min(p.ktm, std::max(0, atoi(ev)) & ~3);
  }
  p.nslot = (int)std::max<size_t>(2, std::min<size_t>(64, (budget - queue_bytes - 4096 - resid_bytes) / slot_bytes));
  // ring + 1 KiB pad (branch-free over-reads past the last column stay in-bounds) + resident k-blocks + row
  // queue + row statistics + barriers + control + reduction scratch
  cfg->smem = (size_t)p.nslot * slot_bytes + 1024 + resid_bytes + queue_bytes + ((size_t)p.nslot + p.qn) * 16 +
              16 + 64 + 128 * 8 + 64;
  p.iters = rows_only ? 1 : iters;
  p.rows_only = rows_only ? 1 : 0;
  p.tol = a.tol;
  p.check_every = a.check_every > 0 ? a.check_every : 1;
  p.partials = ws.partials[parity & 1];
  p.state = ws.state;
  p.plines = ws.plines;
  p.zlines = ws.zlines;
  p.rlines = ws.rlines;
  p.lepoch = ws.lepoch;
  p.lcap = ws.lcap;
  if (!rows_only && (!ws.plines || up.U > ws.lcap)) return cudaErrorInvalidValue;
  p.evict_last_rows = 0;
  p.diag = (int)(a.flags & (COT_DIAG_NO_COMPUTE | COT_DIAG_NO_SYNC | COT_DIAG_NO_STREAM));
  p.pre = (a.flags & COT_PRECOMPUTED) ? 1 : 0;
  if (const char* ev = getenv("COT_EVICT_LAST_ROWS")) p.evict_last_rows = atoi(ev);   // L2 residency experiment
  p.trace = nullptr;
  p.nranks = 0;
  cfg->threads = (p.nk + p.ne + 1) * 32;
  cfg->grid = (int)up.U;
  cfg->cpt = cpt;
  cfg->ept = ept;
  cfg->KS = KS;
  cfg->fn = cfg->fn_emu = nullptr;
#define COT_PICK(C_, E_, K_)                     \
  if (cpt == C_ && ept == E_ && KS == K_) {      \
    cfg->fn = (void*)k_iter_tma<C_, E_, K_>;     \
    cfg->fn_emu = (void*)k_iter_tma_emu<C_, E_, K_>; \
  }
#define COT_PICK_K(C_, E_) \
  COT_PICK(C_, E_, 1) COT_PICK(C_, E_, 2) COT_PICK(C_, E_, 4) COT_PICK(C_, E_, 8) COT_PICK(C_, E_, 16)
  COT_PICK_K(1, 1) COT_PICK_K(1, 2) COT_PICK_K(2, 1)
#undef COT_PICK_K
#undef COT_PICK
  if (!cfg->fn) return cudaErrorInvalidValue;
  return cudaSuccess;
}

cudaError_t check_occupancy(void* fn, int threads, size_t smem, int grid, int sms) {
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  if (grid > occ * sms) return cudaErrorInvalidConfiguration;   // one unit per co-resident CTA
  return cudaSuccess;
}
}  // namespace

namespace {
// Diagnostics (COT_TRACE=1): per-CTA cycle counters of one persistent launch, printed as means / maxima.
unsigned long long* trace_begin(cudaStream_t s) {
  static unsigned long long* trace_buf = nullptr;
  if (!getenv("COT_TRACE")) return nullptr;
  if (!trace_buf) cudaMalloc(&trace_buf, 4096 * 16 * sizeof(unsigned long long));
  cudaMemsetAsync(trace_buf, 0, 4096 * 16 * sizeof(unsigned long long), s);
  return trace_buf;
}
void trace_end(const unsigned long long* trace, int grid, int iters, cudaStream_t s) {
  std::vector<unsigned long long> h((size_t)grid * 16);
  cudaStreamSynchronize(s);
  cudaMemcpy(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost);
  double acc[16] = {0}, mx[16] = {0};
  for (int b = 0; b < grid; ++b)
    for (int k = 0; k < 16; ++k) {
      acc[k] += (double)h[(size_t)b * 16 + k] / grid;
      mx[k] = std::max(mx[k], (double)h[(size_t)b * 16 + k]);
    }
  const double it = iters > 0 ? iters : 1;
  fprintf(stderr,
          "[cot trace] iters=%d per-iter cycles (mean/max over CTAs): prod_wait %.0f/%.0f prod_total %.0f/%.0f "
          "ksum %.0f/%.0f epi_busy %.0f/%.0f epi_wait_z %.0f/%.0f [epi: compute %.0f reduce %.0f; colpass %.0f; "
          "queue wait %.0f/%.0f; ksum queue wait %.0f; colpass poll %.0f; publish %.0f] last epilogue warp: compute "
          "%.0f reduce %.0f busy %.0f wait_z %.0f\n",
          iters, acc[0] / it, mx[0] / it, acc[1] / it, mx[1] / it, acc[3] / it, mx[3] / it, acc[4] / it,
          mx[4] / it, acc[5] / it, mx[5] / it, acc[2] / it, acc[6] / it, acc[7] / it, acc[8] / it, mx[8] / it,
          acc[9] / it, acc[10] / it, acc[11] / it, acc[12] / it, acc[13] / it, acc[14] / it, acc[15] / it);
}
}  // namespace

cudaError_t launch_iter_tma(const IterArgs& a, const Workspace& ws, int iters, bool rows_only, int parity,
                            cudaStream_t s) {
  int sms = device_sm_count();
  if (const char* ev = getenv("COT_MAX_CTAS")) sms = std::max(1, std::min(sms, atoi(ev)));   // experiments
  TmaParams p;
  TmaCfg cfg;
  cudaError_t e = tma_config(a, ws, iters, rows_only, parity, sms, &p, &cfg);
  if (e != cudaSuccess) return e;
  // A stream larger than L2: the first rows of every block (~56 MB of it) are streamed with an L2 evict_last hint
  // and stay resident across iterations, the rest evict_first (C4: rows [0, 244) of the 56 streamed k-blocks;
  // 33.8 -> 32.0 us per iteration; 192-288 rows measured flat, 320 and more thrash). COT_EVICT_LAST_ROWS overrides.
  // Rows-only launches (cerot_iter_sharded's row pass, replayed once per iteration) use the same split: L2
  // keeps its contents across launches, so the evict_last rows are re-read from L2 by the next launch.
  if ((rows_only || iters > 1) && !getenv("COT_EVICT_LAST_ROWS")) {
    const double row_bytes = (double)(a.n - p.kres - p.ktm) * (double)a.m * 4.0;   // one row's streamed k-blocks
    if (row_bytes > 0.0 && row_bytes * (double)a.R > 96e6)
      p.evict_last_rows = (int)std::min<double>((double)a.R, (rows_only ? 40e6 : 56e6) / row_bytes);
  }   // rows-only C4 (whole rows streamed): 0 / 150 / 213 / 300 rows measured 52.5 / 50.8 / 52.5 / 52.4 us/iter
  p.trace = trace_begin(s);
  e = check_occupancy(cfg.fn, cfg.threads, cfg.smem, cfg.grid, sms);
  if (e != cudaSuccess) return e;
  const int grid = cfg.grid;
  void* args[] = {&p};
  if (rows_only) return cudaLaunchKernel(cfg.fn, dim3(grid), dim3(cfg.threads), args, cfg.smem, s);
  e = cudaLaunchCooperativeKernel(cfg.fn, dim3(grid), dim3(cfg.threads), args, cfg.smem, s);
  if (e == cudaSuccess && p.trace) trace_end(p.trace, grid, iters, s);
  return e;
}

int fused_column_slices(int64_t m, int nranks, int sms) {
  // the smallest unit count of a balanced row partition (rows per rank = floor or ceil of m / nranks)
  const int64_t lo = m / nranks, hi = (m + nranks - 1) / nranks;
  int64_t ncs = unit_plan(1, hi, sms).U;
  if (lo >= 1) ncs = std::min<int64_t>(ncs, unit_plan(1, lo, sms).U);
  return (int)ncs;
}

cudaError_t launch_iter_tma_fused(const FusedRank* r, int nv, int nranks, bool emulate, int iters, cudaStream_t s) {
  if (nv < 1 || nv > kMaxRanks || nranks < 1 || nranks > kMaxRanks || (emulate && nv != nranks) ||
      (!emulate && nv != 1))
    return cudaErrorInvalidValue;
  const int sms_dev = device_sm_count();
  int sms = emulate ? sms_dev / nranks : sms_dev;   // emulation: each virtual rank gets 1/nranks of the SMs
  if (const char* ev = getenv("COT_MAX_CTAS")) sms = std::max(1, std::min(sms, atoi(ev)));   // experiments
  if (sms < 1) return cudaErrorInvalidConfiguration;
  TmaMulti pm;
  memset(&pm, 0, sizeof(pm));
  TmaCfg cfg0;
  // column slices: identical on every rank (nranks == 1: any row range, the slices of this launch)
  int ncs = emulate || nranks == 1 ? 1 << 30 : fused_column_slices(r[0].a.m, nranks, sms);
  size_t smem = 0;
  pm.nv = nv;
  pm.base[0] = 0;
  for (int v = 0; v < nv; ++v) {
    TmaCfg cfg;
    cudaError_t e = tma_config(r[v].a, r[v].ws, iters, false, 0, sms, &pm.rp[v], &cfg);
    if (e != cudaSuccess) return e;
    if (v == 0) cfg0 = cfg;
    if (cfg.fn != cfg0.fn || cfg.threads != cfg0.threads) return cudaErrorInvalidValue;   // same instance
    smem = std::max(smem, cfg.smem);
    pm.base[v + 1] = pm.base[v] + cfg.grid;
    if (emulate || nranks == 1) ncs = std::min(ncs, cfg.grid);
    else if (cfg.grid < ncs) return cudaErrorInvalidValue;   // the caller's rows are not a balanced partition
    TmaParams& p = pm.rp[v];
    p.nranks = nranks;
    p.rank = r[v].rank;
    for (int q = 0; q < nranks; ++q) p.xpeer[q] = r[v].xpeer[q];
    p.xepoch = r[v].xepoch;
    // a shard whose cost rows fit comfortably in L2 is kept there across iterations
    if (!emulate && (double)(r[v].a.n + 1) * r[v].a.R * r[v].a.m * 4.0 <= 80e6) p.evict_last_rows = (int)r[v].a.R;
    // emulated ranks share one GPU's L2: the unsharded launch's ~56 MB evict_last budget split over them (C4, 8
    // virtual ranks: 16 / 27 / 40 rows each measured 39.9 / 39.9 / 44.2 us per iteration against 41.3 with none)
    // (1/2/4 virtual ranks then match the unsharded launch: 31.8 / 31.9 / 32.3 vs 32.0; 8: 40.0). A real rank
    // whose shard does not fit L2 takes the unsharded launch's rule (the first ~56 MB of rows evict_last).
    if (!getenv("COT_EVICT_LAST_ROWS") && p.evict_last_rows < (int)r[v].a.R) {
      const double row_bytes = (double)(r[v].a.n - p.kres - p.ktm) * (double)r[v].a.m * 4.0;
      const double budget = emulate ? 40e6 / nranks : 56e6;
      if (row_bytes > 0.0 && row_bytes * (double)r[v].a.R * (emulate ? nranks : 1) > 96e6)
        p.evict_last_rows = (int)std::min<double>((double)r[v].a.R, budget / row_bytes);
    }
  }
  for (int v = 0; v < nv; ++v) pm.rp[v].ncs = ncs;
  const int grid = pm.base[nv];
  if (!emulate) {
    cudaError_t e = check_occupancy(cfg0.fn, cfg0.threads, smem, grid, sms_dev);
    if (e != cudaSuccess) return e;
    pm.rp[0].trace = trace_begin(s);
    void* args[] = {&pm.rp[0]};
    e = cudaLaunchCooperativeKernel(cfg0.fn, dim3(grid), dim3(cfg0.threads), args, smem, s);
    if (e == cudaSuccess && pm.rp[0].trace) trace_end(pm.rp[0].trace, grid, iters, s);
    return e;
  }
  cudaError_t e = check_occupancy(cfg0.fn_emu, cfg0.threads, smem, grid, sms_dev);
  if (e != cudaSuccess) return e;
  void* args[] = {&pm};
  return cudaLaunchCooperativeKernel(cfg0.fn_emu, dim3(grid), dim3(cfg0.threads), args, smem, s);
}

}  // namespace cot
