// K-ITER-RES: the cyclic Sinkhorn iteration (Alg. 2 lines 4-5; log domain of eq. P:403-411) for a
// problem -- or one GPU's row shard of it -- whose n*R*m fp32 cost values fit ON CHIP: in the tensor memory
// (TMEM, 256 KB per SM, used here as a per-thread store of cost values) plus shared memory of one CTA per SM.
// The cost is loaded once per launch; every iteration still evaluates all n*R*m Gibbs terms
// s'_ij = sum_k 2^{a_ij - C_ijk log2e/eps} (a_ij = round(G_ij log2e/eps)), now from on-chip memory, so the
// per-iteration bound is the SFU (MUFU.EX2), not HBM. Serves C3 (n = 4, m = 1024: 16 MiB) and the C4 row
// shards of 4- and 8-GPU partitions (32 / 64 MiB per GPU), which the streaming kernel (k_iter_tma.cu) can
// only serve from L2 at a per-row pipeline cost.
//
// Work split: each row of the shard is cut into h pieces of W = m/h consecutive columns (h = 1, 2 or 4); the
// h pieces of a row live in the h CTAs of one thread-block cluster (CTA rank q holds columns [qW, (q+1)W)),
// rows are spread over the ncl clusters in contiguous balanced ranges. A CTA's "quads" (one row piece x four
// consecutive columns, all n k-blocks) are its work items.
//
//   k-sum warps (8): s'_ij of every quad of the CTA for iteration t+1 while the epilogue still works on t
//     (the k-sums do not depend on the potentials), double-buffered in shared memory (mbarriers); throttled to
//     start when iteration t's reduction is issued when they are short. Quad Q of thread kt = Q % 256 sits in
//     the thread's TMEM column range (tcgen05.ld) while it has room, else in shared memory, else (a shard
//     slightly over the capacity) it is streamed from L2 every iteration.
//   epilogue warps (8), per iteration:
//     row pass: t'_ij = s'_ij 2^{kz_j - a_ij - kM} Fz_j with an exact per-warp shift kM (integer maximum, one
//       REDUX), piece sums combined with exact power-of-two rescaling (one warp per row); with h > 1 the
//       pieces' (sum, shift) pairs go to every CTA of the cluster with st.async + the receiver's mbarrier
//       transaction count, so all h CTAs hold the identical row sum r_i and shift kM_i;
//     column pass: P_j = sum_i (alpha_i / r_i) t_ij over the CTA's rows, converted to 64-bit unsigned fixed
//       point (scale 2^S, 2^(53-S) >= sum alpha: every column sum fits below the count byte) and added with
//       coalesced red.global.add.u64 into the iteration's column sums -- integer addition, so the sums do not
//       depend on the order in which CTAs (or ranks) arrive: deterministic, and bitwise the same on every rank;
//     device-wide step, one GPU: one cumulative arrival counter per column group (the CTAs holding the same
//       columns), then every CTA reads its W column sums;
//     device-wide step, sharded (cerot_iter_fused): every partial carries 1 in its top byte, so the rank-local
//       sum of a column counts its contributions; the owner of each 1/ncl column slice polls its columns until
//       the count is ncl, pushes the sums (again with 1 in the top byte) into every rank's exchange sums with
//       system-scope reductions and zeroes its rank-local slot; every CTA polls its W exchange columns until
//       their count is nranks. No fence, counter or CTA barrier after the reductions.
//     q-update (every CTA of a group, same bits): 2^{kz_j} Fz_j <- 2^{kz_j} Fz_j beta_j / c_j, renormalised from
//       the exponent bits (no log / exp per column); the freeze-rule monitor n sum_j |c_j - beta_j| is formed by
//       every CTA from all m sums in a fixed order on the iterations that need it.
//   Sum buffers rotate over three slots by the absolute reduction index (workspace / exchange epochs); slots
//   are zeroed by their owners after the last read (no per-iteration memset, no grid barrier).
#include "common.cuh"
#include "internal.h"

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <vector>

namespace cot {

constexpr int kResNK = 8;                          // k-sum warps (TMEM: two warps per 32-lane quarter)
constexpr int kResNE = 8;                          // epilogue warps
constexpr int kResThreads = (kResNK + kResNE) * 32;
constexpr int kResKT = kResNK * 32;                // k-sum threads
constexpr int kResET = kResNE * 32;                // epilogue threads
constexpr int kResMaxSmem = 227 * 1024;
enum { RCTL_TBASE = 0, RCTL_HALT = 1, RCTL_TIMEOUT = 2 };

struct ResParams {
  const float* C;        // [n][R][m] (this rank's rows)
  const float* G;        // [R][m]
  const double* alpha;   // [m] (global row index)
  const double* beta;    // [m]
  double* w_hat;         // [m]
  double* z_hat;         // [m]
  const double* eps;     // [1]
  int n, m, R, row_begin;
  int h, W, ncl;         // pieces per row (= cluster size), piece width, clusters of this rank
  int MR, nq_max;        // max rows per cluster, max quads per CTA
  int tq, nsq;           // quads per k-sum thread held in TMEM, shared-memory quad slots
  int throttle;          // k-sums of iteration t start while t - 1 is reduced (else as soon as a buffer is free)
  int iters;
  double tol;
  long long check_every;
  SolverState* state;
  unsigned long long* lsum;    // [3][m] rank-local column sums (workspace)
  unsigned* lcnt;              // [8] arrival counters per column group; [8..9]: reduction epoch (u64)
  int nranks, rank;            // nranks == 0: no cross-rank level
  unsigned long long* xsum[kMaxRanks];   // rank r's [3][m] exchange sums, as addressed by this rank
  unsigned* xcnt[kMaxRanks];             // rank r's [8] exchange counters; [8..9]: exchange epoch
  unsigned long long* trace;
};
struct ResMulti {
  ResParams rp[kMaxRanks];
  int base[kMaxRanks + 1];
  int nv;
};

struct ResLayout {
  size_t scost, sbuf, ash, zf, bet, zk, colbuf, rowf, rowr, rowk, lal, alph, chunk, rx, red, bars, ctl, total;
};
__host__ __device__ inline size_t res_take(size_t& o, size_t bytes) {
  const size_t r = o;
  o = (o + bytes + 15) & ~(size_t)15;
  return r;
}
__host__ __device__ inline ResLayout res_layout(int n, int nsq, int nq_max, int W, int MR, int h) {
  ResLayout L;
  size_t o = 0;
  L.scost = res_take(o, (size_t)n * nsq * 16);   // [n][nsq] float4
  L.sbuf = res_take(o, (size_t)2 * nq_max * 16);  // [2][nq_max] float4: s'
  L.ash = res_take(o, (size_t)nq_max * 16);       // [nq_max] int4: a_ij
  L.zf = res_take(o, (size_t)W * 8);              // Fz_j (z_j log2e = kz_j + log2 Fz_j)
  L.bet = res_take(o, (size_t)W * 8);             // beta_j
  L.zk = res_take(o, (size_t)W * 4);              // kz_j
  L.colbuf = res_take(o, (size_t)W * 8);          // fixed-point column partials of the CTA (bulk-reduced)
  L.rowf = res_take(o, (size_t)2 * MR * 8);       // [2][MR] alpha_i / r_i
  L.rowr = res_take(o, (size_t)2 * MR * 8);       // [2][MR] r_i (relative to 2^kM_i)
  L.rowk = res_take(o, (size_t)2 * MR * 4);       // [2][MR] kM_i
  L.lal = res_take(o, (size_t)MR * 8);            // log alpha_i
  L.alph = res_take(o, (size_t)MR * 8);           // alpha_i
  L.chunk = res_take(o, (size_t)(nq_max / 32 + 1) * 16);   // per-32-quad (sum, shift)
  L.rx = res_take(o, (size_t)2 * MR * h * 16);    // [2][MR][h] (piece sum, shift) from every cluster CTA
  L.red = res_take(o, 64 * 8);
  L.bars = res_take(o, 8 * 8);
  L.ctl = res_take(o, 16 * 4);
  L.total = o;
  return L;
}

// ------------------------------------------------------------------------------------------ device helpers
#define COT_TLD16(taddr, r)                                                                                      \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"  \
               " [%16];"                                                                                         \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),  \
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),        \
                 "=r"(r[15])                                                                                     \
               : "r"(taddr))
#define COT_TST16(taddr, r)                                                                                     \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"   \
               "%15,%16};" ::"r"(taddr),                                                                        \
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), \
               "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]))

__device__ __forceinline__ void ebar() { asm volatile("bar.sync 1, %0;" ::"r"(kResET) : "memory"); }
__device__ __forceinline__ void kbar() { asm volatile("bar.sync 2, %0;" ::"r"(kResKT) : "memory"); }
__device__ __forceinline__ unsigned long long res_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr unsigned long long kResTimeoutNs = 20000000000ull;   // 20 s without an arrival: give up (COT_E_PEER)
// 2^k for an integer k <= 0 (0 below the normal range: such a partial is negligible next to the maximum's)
__device__ __forceinline__ double pow2i(int k) { return k < -1022 ? 0.0 : __hiloint2double((k + 1023) << 20, 0); }
__device__ __forceinline__ void red_add_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned cluster_map(unsigned saddr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// spin until the cumulative counter reaches `want` (wrap-safe); false after the timeout
__device__ __forceinline__ bool wait_count(const unsigned* c, unsigned want) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
  if ((int)(v - want) >= 0) return true;
  const unsigned long long t0 = res_timer();
  while (true) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
    if ((int)(v - want) >= 0) return true;
    if (res_timer() - t0 > kResTimeoutNs) return false;
  }
}
// Exchange sums (multi-GPU level): value in the low 56 bits, contribution count in the top byte.
constexpr unsigned long long kCntOne = 1ull << 56;
constexpr unsigned long long kValMask = kCntOne - 1ull;
// the exchange sums are self-validating (count byte): a relaxed load of this GPU's own memory is enough
__device__ __forceinline__ unsigned long long ld_poll(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// one column sum polled until its count is `want` (acquire: the sum's contributions are then all visible)
__device__ __forceinline__ bool poll_sum1(const unsigned long long* p, unsigned want, unsigned long long& v) {
  unsigned long long t0 = 0;
  while (true) {
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    if ((unsigned)(v >> 56) == want) return true;
    if (t0 == 0) t0 = res_timer();
    else if (res_timer() - t0 > kResTimeoutNs) return false;
  }
}
// the thread's columns j = et + k * kResET < W (k < 4), polled together until every count is `want`
__device__ __forceinline__ bool poll_sums4(const unsigned long long* base, int et, int W, unsigned want,
                                           unsigned long long (&v)[4]) {
  unsigned todo = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (et + k * kResET < W) todo |= 1u << k;
  unsigned long long t0 = 0;
  while (true) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (todo & (1u << k)) v[k] = ld_poll(base + et + k * kResET);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if ((todo & (1u << k)) && (unsigned)(v[k] >> 56) == want) todo &= ~(1u << k);
    if (!todo) return true;
    if (t0 == 0) t0 = res_timer();
    else if (res_timer() - t0 > kResTimeoutNs) return false;
  }
}
// OR of a predicate over the epilogue threads (a barrier itself)
__device__ __forceinline__ bool bar_or(bool v) {
  unsigned r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\tbar.red.or.pred q, 1, %2, p;\n\tselp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"((unsigned)v), "r"(kResET)
      : "memory");
  return r != 0;
}

// F = Fz 2^e with Fz in [2^-1/2, 2^1/2) (exact: exponent bits only); k += e. F positive and normal.
__device__ __forceinline__ double renorm_pow2(double F, int& k) {
  const int hi = __double2hiint(F);
  int e = ((hi >> 20) & 0x7ff) - 1023;
  double M = __hiloint2double((hi & 0x000FFFFF) | 0x3FF00000, __double2loint(F));
  if (M >= 1.4142135623730951) {
    M *= 0.5;
    e += 1;
  }
  k += e;
  return M;
}

__device__ __forceinline__ void res_body(const ResParams& p, const int b) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = p.h, W = p.W, m = p.m, n = p.n, W4 = W / 4, MR = p.MR, nqmax = p.nq_max;
  const int c = b / h, q = b % h;                         // cluster (row range), piece (column group)
  const int lr0 = (int)((long long)c * p.R / p.ncl), lr1 = (int)((long long)(c + 1) * p.R / p.ncl);
  const int nrows = lr1 - lr0, nq = nrows * W4;
  const int col0 = q * W;
  const ResLayout L = res_layout(n, p.nsq, nqmax, W, MR, h);
  float4* scost = reinterpret_cast<float4*>(smem + L.scost);
  float4* sbuf = reinterpret_cast<float4*>(smem + L.sbuf);
  int4* ash = reinterpret_cast<int4*>(smem + L.ash);
  double* zf = reinterpret_cast<double*>(smem + L.zf);
  double* bet = reinterpret_cast<double*>(smem + L.bet);
  int* zk = reinterpret_cast<int*>(smem + L.zk);
  unsigned long long* colbuf = reinterpret_cast<unsigned long long*>(smem + L.colbuf);
  double* rowf = reinterpret_cast<double*>(smem + L.rowf);
  double* rowr = reinterpret_cast<double*>(smem + L.rowr);
  int* rowk = reinterpret_cast<int*>(smem + L.rowk);
  double* lal = reinterpret_cast<double*>(smem + L.lal);
  double* alph = reinterpret_cast<double*>(smem + L.alph);
  double2* chunk = reinterpret_cast<double2*>(smem + L.chunk);
  double2* rx = reinterpret_cast<double2*>(smem + L.rx);
  double* red = reinterpret_cast<double*>(smem + L.red);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* sfull = bars;        // [2] k-sums of an iteration written (one arrival per k-sum warp)
  uint64_t* sgo = bars + 2;      // the epilogue has issued an iteration's reduction: the next k-sums may start
  uint64_t* sempty = bars + 5;   // [2] the epilogue has finished with an s' buffer
  uint64_t* rbar = bars + 4;     // row-piece sums of the cluster arrived (h arrivals per iteration)
  unsigned* ctl = reinterpret_cast<unsigned*>(smem + L.ctl);

  const float c2 = (float)(COT_LOG2E / p.eps[0]);
  const bool active0 = p.state[0].active != 0;
  if (threadIdx.x == 0) {
    mbar_init(&sfull[0], kResNK);
    mbar_init(&sfull[1], kResNK);
    mbar_init(sgo, 1);
    mbar_init(&sempty[0], 1);
    mbar_init(&sempty[1], 1);
    mbar_init(rbar, 1);
    for (int k = 0; k < 16; ++k) ctl[k] = 0;
    fence_mbar_init();
  }
  // a_ij = round(G_ij log2e/eps) of every quad (the k-sum warps' exact shift; fp32 as in k_iter_tma)
  for (int Q = threadIdx.x; Q < nq; Q += kResThreads) {
    const int lr = Q / W4, cq = Q - lr * W4;
    const float4 g4 = __ldg(reinterpret_cast<const float4*>(p.G + (size_t)(lr0 + lr) * m + col0) + cq);
    ash[Q] = make_int4(__float2int_rn(g4.x * c2), __float2int_rn(g4.y * c2), __float2int_rn(g4.z * c2),
                       __float2int_rn(g4.w * c2));
  }
  // shared-memory quads: [k][nsq] float4, quad Q = 256 tq + sq
  const int nsq_used = min(p.nsq, max(0, nq - kResKT * p.tq));   // the rest (if any) is streamed from L2
  for (int idx = threadIdx.x; idx < nsq_used * n; idx += kResThreads) {
    const int k = idx / nsq_used, sq = idx - k * nsq_used;
    const int Q = kResKT * p.tq + sq, lr = Q / W4, cq = Q - lr * W4;
    scost[(size_t)k * p.nsq + sq] =
        __ldg(reinterpret_cast<const float4*>(p.C + ((size_t)k * p.R + lr0 + lr) * m + col0) + cq);
  }
  if (warp == 0 && p.tq > 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&ctl[RCTL_TBASE])));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (h > 1) cluster_sync_all();   // the peers' mbarriers are initialised before any remote arrival

  if (warp < kResNK) {
    // =========================================================================== k-sum warps
    const int kt = threadIdx.x;
    const unsigned tbase = ctl[RCTL_TBASE];
    const unsigned ta = tbase + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)((warp >> 2) * 256);
    const int nt = min(p.tq, (nq - kt + kResKT - 1) / kResKT);   // this thread's TMEM quads (warp-uniform: nq % 32 == 0)
    // load the thread's TMEM quads once per launch: words (k, v) of quad s at columns s*4n + 4k + v
    for (int s = 0; s < nt; ++s) {
      const int Q = kt + kResKT * s, lr = Q / W4, cq = Q - lr * W4;
      const float4* src = reinterpret_cast<const float4*>(p.C + ((size_t)lr0 + lr) * m + col0) + cq;
      for (int k0 = 0; k0 < n; k0 += 4) {
        unsigned r[16];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const float4 v = k0 + kk < n ? __ldg(src + (size_t)(k0 + kk) * p.R * (m / 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
          r[4 * kk] = __float_as_uint(v.x);
          r[4 * kk + 1] = __float_as_uint(v.y);
          r[4 * kk + 2] = __float_as_uint(v.z);
          r[4 * kk + 3] = __float_as_uint(v.w);
        }
        COT_TST16(ta + (unsigned)(s * 4 * n + 4 * k0), r);
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    long long tk_wait = 0, tk_busy = 0;
    for (int t = 0; active0 && t < p.iters; ++t) {
      const int buf = t & 1;
      const long long tk0 = p.trace ? clock64() : 0;
      // throttled (k-sums shorter than the device-wide step): start once iteration t - 1 is being reduced, so the
      // k-sums fill that wait instead of competing with the epilogue's passes; otherwise as soon as the buffer of
      // iteration t - 2 is free. A halted epilogue never signals.
      if (p.throttle ? t >= 1 : t >= 2) {
        const uint32_t par = p.throttle ? (uint32_t)(t - 1) & 1u : (uint32_t)((t - 2) >> 1) & 1u;
        uint64_t* wb = p.throttle ? sgo : &sempty[buf];
        bool halt = false;
        while (true) {
          uint32_t ok;
          asm volatile(
              "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
              "selp.u32 %0, 1, 0, p;\n\t}"
              : "=r"(ok)
              : "r"(smem_u32(wb)), "r"(par)
              : "memory");
          if (ok) break;
          if (*(volatile unsigned*)&ctl[RCTL_HALT]) {
            halt = true;
            break;
          }
        }
        if (__any_sync(0xffffffffu, halt)) break;
      }
      const long long tk1 = p.trace ? clock64() : 0;
      float4* out = sbuf + (size_t)buf * nqmax;
      // TMEM quads: 8 k-rows (two x16 loads) per wait
      for (int s = 0; s < nt; ++s) {
        const int Q = kt + kResKT * s;
        const int4 a4 = ash[Q];
        const float g0 = (float)a4.x, g1 = (float)a4.y, g2 = (float)a4.z, g3 = (float)a4.w;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
        const unsigned tq0 = ta + (unsigned)(s * 4 * n);
        int k0 = 0;
        for (; k0 + 8 <= n; k0 += 8) {
          unsigned x[16], y[16];
          COT_TLD16(tq0 + 4 * k0, x);
          COT_TLD16(tq0 + 4 * k0 + 16, y);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          float e[32];
#pragma unroll
          for (int w = 0; w < 16; w += 4) {
            e[w] = ex2(fmaf(-__uint_as_float(x[w]), c2, g0));
            e[w + 1] = ex2(fmaf(-__uint_as_float(x[w + 1]), c2, g1));
            e[w + 2] = ex2(fmaf(-__uint_as_float(x[w + 2]), c2, g2));
            e[w + 3] = ex2(fmaf(-__uint_as_float(x[w + 3]), c2, g3));
            e[16 + w] = ex2(fmaf(-__uint_as_float(y[w]), c2, g0));
            e[16 + w + 1] = ex2(fmaf(-__uint_as_float(y[w + 1]), c2, g1));
            e[16 + w + 2] = ex2(fmaf(-__uint_as_float(y[w + 2]), c2, g2));
            e[16 + w + 3] = ex2(fmaf(-__uint_as_float(y[w + 3]), c2, g3));
          }
          s0 += ((e[0] + e[4]) + (e[8] + e[12])) + ((e[16] + e[20]) + (e[24] + e[28]));
          s1 += ((e[1] + e[5]) + (e[9] + e[13])) + ((e[17] + e[21]) + (e[25] + e[29]));
          s2 += ((e[2] + e[6]) + (e[10] + e[14])) + ((e[18] + e[22]) + (e[26] + e[30]));
          s3 += ((e[3] + e[7]) + (e[11] + e[15])) + ((e[19] + e[23]) + (e[27] + e[31]));
        }
        if (k0 < n) {   // n % 8 == 4 (n % 4 == 0 for TMEM placement)
          unsigned x[16];
          COT_TLD16(tq0 + 4 * k0, x);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          s0 += (ex2(fmaf(-__uint_as_float(x[0]), c2, g0)) + ex2(fmaf(-__uint_as_float(x[4]), c2, g0))) +
                (ex2(fmaf(-__uint_as_float(x[8]), c2, g0)) + ex2(fmaf(-__uint_as_float(x[12]), c2, g0)));
          s1 += (ex2(fmaf(-__uint_as_float(x[1]), c2, g1)) + ex2(fmaf(-__uint_as_float(x[5]), c2, g1))) +
                (ex2(fmaf(-__uint_as_float(x[9]), c2, g1)) + ex2(fmaf(-__uint_as_float(x[13]), c2, g1)));
          s2 += (ex2(fmaf(-__uint_as_float(x[2]), c2, g2)) + ex2(fmaf(-__uint_as_float(x[6]), c2, g2))) +
                (ex2(fmaf(-__uint_as_float(x[10]), c2, g2)) + ex2(fmaf(-__uint_as_float(x[14]), c2, g2)));
          s3 += (ex2(fmaf(-__uint_as_float(x[3]), c2, g3)) + ex2(fmaf(-__uint_as_float(x[7]), c2, g3))) +
                (ex2(fmaf(-__uint_as_float(x[11]), c2, g3)) + ex2(fmaf(-__uint_as_float(x[15]), c2, g3)));
        }
        out[Q] = make_float4(s0, s1, s2, s3);
      }
      // quads beyond the on-chip capacity (streamed from L2 every iteration: a shard that does not quite fit, the
      // 4-GPU C4 shard): the k-blocks of each such quad are split over 4 consecutive lanes (16 k-rows each at
      // n = 64, eight loads in flight per lane) so the loads' latency is paid in parallel, and the four parts are
      // combined by a fixed shuffle tree
      {
        const int qs0 = kResKT * p.tq + p.nsq;   // first streamed quad
        const int items = max(0, nq - qs0) * 4;
        const int kc = (n + 3) / 4;              // k-rows per part
        const size_t ks = (size_t)p.R * (m / 4);
        for (int base = 0; base < items; base += kResKT) {   // the same trip count in every k-sum warp
          const int it = base + kt;
          const int Q = qs0 + (it >> 2);
          float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
          if (it < items) {
            const int kb = (it & 3) * kc, ke = min(n, kb + kc);
            const int lr = Q / W4, cq = Q - lr * W4;
            const float4* src = reinterpret_cast<const float4*>(p.C + ((size_t)lr0 + lr) * m + col0) + cq;
            const int4 a4 = ash[Q];
            const float g0 = (float)a4.x, g1 = (float)a4.y, g2 = (float)a4.z, g3 = (float)a4.w;
            float4 A[8], Bn[8];
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              A[kk] = kb + kk < ke ? __ldcg(src + (size_t)(kb + kk) * ks) : make_float4(0.f, 0.f, 0.f, 0.f);
            for (int k0 = kb; k0 < ke; k0 += 8) {
#pragma unroll
              for (int kk = 0; kk < 8; ++kk)
                Bn[kk] = k0 + 8 + kk < ke ? __ldcg(src + (size_t)(k0 + 8 + kk) * ks) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
              for (int kk = 0; kk < 8; ++kk)
                if (k0 + kk < ke) {
                  s0 += ex2(fmaf(-A[kk].x, c2, g0));
                  s1 += ex2(fmaf(-A[kk].y, c2, g1));
                  s2 += ex2(fmaf(-A[kk].z, c2, g2));
                  s3 += ex2(fmaf(-A[kk].w, c2, g3));
                }
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) A[kk] = Bn[kk];
            }
          }
#pragma unroll
          for (int o = 1; o <= 2; o <<= 1) {
            s0 += __shfl_xor_sync(0xffffffffu, s0, o);
            s1 += __shfl_xor_sync(0xffffffffu, s1, o);
            s2 += __shfl_xor_sync(0xffffffffu, s2, o);
            s3 += __shfl_xor_sync(0xffffffffu, s3, o);
          }
          if (it < items && (it & 3) == 0) out[Q] = make_float4(s0, s1, s2, s3);
        }
      }
      // shared-memory quads: four k-rows per step, loads first
      for (int Q = kt + kResKT * nt; Q < nq; Q += kResKT) {
        const int sq = Q - kResKT * p.tq;
        if (sq >= p.nsq) break;   // streamed (above)
        const int4 a4 = ash[Q];
        const float g0 = (float)a4.x, g1 = (float)a4.y, g2 = (float)a4.z, g3 = (float)a4.w;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
        const float4* cb = scost + sq;
        int k = 0;
        for (; k + 4 <= n; k += 4) {
          const float4 x0 = cb[(size_t)k * p.nsq], x1 = cb[(size_t)(k + 1) * p.nsq];
          const float4 x2 = cb[(size_t)(k + 2) * p.nsq], x3 = cb[(size_t)(k + 3) * p.nsq];
          s0 += (ex2(fmaf(-x0.x, c2, g0)) + ex2(fmaf(-x1.x, c2, g0))) + (ex2(fmaf(-x2.x, c2, g0)) + ex2(fmaf(-x3.x, c2, g0)));
          s1 += (ex2(fmaf(-x0.y, c2, g1)) + ex2(fmaf(-x1.y, c2, g1))) + (ex2(fmaf(-x2.y, c2, g1)) + ex2(fmaf(-x3.y, c2, g1)));
          s2 += (ex2(fmaf(-x0.z, c2, g2)) + ex2(fmaf(-x1.z, c2, g2))) + (ex2(fmaf(-x2.z, c2, g2)) + ex2(fmaf(-x3.z, c2, g2)));
          s3 += (ex2(fmaf(-x0.w, c2, g3)) + ex2(fmaf(-x1.w, c2, g3))) + (ex2(fmaf(-x2.w, c2, g3)) + ex2(fmaf(-x3.w, c2, g3)));
        }
        for (; k < n; ++k) {
          const float4 x0 = cb[(size_t)k * p.nsq];
          s0 += ex2(fmaf(-x0.x, c2, g0));
          s1 += ex2(fmaf(-x0.y, c2, g1));
          s2 += ex2(fmaf(-x0.z, c2, g2));
          s3 += ex2(fmaf(-x0.w, c2, g3));
        }
        out[Q] = make_float4(s0, s1, s2, s3);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sfull[buf]);
      if (p.trace) {
        tk_wait += tk1 - tk0;
        tk_busy += clock64() - tk1;
      }
    }
    if (p.trace && kt == 0) {
      p.trace[(size_t)blockIdx.x * 16 + 0] = tk_wait;
      p.trace[(size_t)blockIdx.x * 16 + 1] = tk_busy;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    kbar();
    if (warp == 0 && p.tq > 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
  } else {
    // =========================================================================== epilogue warps
    const int et = threadIdx.x - kResKT, ew = et >> 5;
    const int nr = p.nranks;
    const bool fused = nr > 0;
    const int slice = (W + p.ncl - 1) / p.ncl;             // columns of the group zeroed / pushed by this CTA
    const int js0 = min(W, c * slice), js1 = min(W, js0 + slice);
    const unsigned long long Er = *reinterpret_cast<volatile unsigned long long*>(p.lcnt + 8);
    const unsigned long long Ex = fused ? *reinterpret_cast<volatile unsigned long long*>(p.xcnt[p.rank] + 8) : 0ull;
    // per-launch setup: own columns' z, beta; own rows' alpha; the fixed-point scale from sum(alpha)
    for (int j = et; j < W; j += kResET) {
      bet[j] = p.beta[col0 + j];
      int k;
      zf[j] = split_z(__ldcg(p.z_hat + col0 + j), k);
      zk[j] = k;
    }
    for (int lr = et; lr < nrows; lr += kResET) {
      const double a = p.alpha[p.row_begin + lr0 + lr];
      alph[lr] = a;
      lal[lr] = log(a);
    }
    double asum = 0.0;
    for (int i = et; i < m; i += kResET) asum += p.alpha[i];
    asum = warp_sum(asum);
    if (lane == 0) red[ew] = asum;
    ebar();
    asum = ((red[0] + red[1]) + (red[2] + red[3])) + ((red[4] + red[5]) + (red[6] + red[7]));
    int ea;
    frexp(asum, &ea);   // sum alpha <= 2^ea: every column sum (<= sum alpha) stays below 2^53 < 2^56 (count byte)
    const int S = 53 - ea;
    const double scale = ldexp(1.0, S), iscale = ldexp(1.0, -S);
    ebar();
    SolverState st = p.state[0];
    const long long iters0 = st.iters;
    bool halted = false, timeout = false, underflow = false;
    const int lpp = min(W4, kResET);            // threads per piece in the row pass
    const int ppr = kResET / lpp;               // pieces per round
    const int cpp = lpp / 32;                   // warp partials (chunks) per piece
    long long tr[7] = {0, 0, 0, 0, 0, 0, 0};   // diagnostics (COT_TRACE): cycles per phase
    int done = 0;
    unsigned long long* lsum = p.lsum;
    unsigned long long* xown = fused ? p.xsum[p.rank] : nullptr;
    for (int t = 0; active0 && t < p.iters; ++t) {
      const int buf = t & 1;
      const unsigned long long T = Er + (unsigned long long)t, TX = Ex + (unsigned long long)t;
      const int sT = (int)(T % 3ull), sTp = (int)((T + 2ull) % 3ull);
      const int sX = (int)(TX % 3ull), sXp = (int)((TX + 2ull) % 3ull);
      long long tp = p.trace ? clock64() : 0;
      auto mark = [&](int slot) {
        if (p.trace) {
          const long long now = clock64();
          tr[slot] += now - tp;
          tp = now;
        }
      };
      if (h > 1 && et == 0) mbar_arrive_expect_tx(rbar, (uint32_t)(h * nrows * 16));
      mbar_wait(&sfull[buf], (uint32_t)(t >> 1) & 1u);
      mark(0);
      const float4* sb = sbuf + (size_t)buf * nqmax;
      // ---- row pass: a warp takes 32 quads of one piece; their terms are summed against the warp's exact maximum
      // exponent (one REDUX), then one warp sum per (warp, piece); RB rounds of pieces in flight per thread
      // RB rounds of pieces in flight per thread: 1 when the CTA has one round (no idle REDUX / shuffles), else 4
      auto row_pass = [&](auto rbc) {
        constexpr int RB = decltype(rbc)::value;
        for (int r0 = 0; r0 * ppr < nrows; r0 += RB) {
          int e[RB][4];
          float4 s4[RB];
          int mxw[RB];
          double v[RB];
          const int cq = et % lpp;
#pragma unroll
          for (int u = 0; u < RB; ++u) {
            const int lr = (r0 + u) * ppr + et / lpp;   // warp-uniform (lpp >= 32)
            int emax = INT_MIN;
            if (lr < nrows) {
              const int Q = lr * W4 + cq;
              s4[u] = sb[Q];
              const int4 a4 = ash[Q];
              const int4 k4 = reinterpret_cast<const int4*>(zk)[cq];
              e[u][0] = k4.x - a4.x;
              e[u][1] = k4.y - a4.y;
              e[u][2] = k4.z - a4.z;
              e[u][3] = k4.w - a4.w;
              emax = max(max(e[u][0], e[u][1]), max(e[u][2], e[u][3]));
            }
            mxw[u] = __reduce_max_sync(0xffffffffu, emax);
          }
          const double2 fa = reinterpret_cast<const double2*>(zf)[2 * cq];
          const double2 fb = reinterpret_cast<const double2*>(zf)[2 * cq + 1];
#pragma unroll
          for (int u = 0; u < RB; ++u) {
            const int lr = (r0 + u) * ppr + et / lpp;
            v[u] = lr < nrows ? (ldexp_pos(s4[u].x, e[u][0] - mxw[u]) * fa.x + ldexp_pos(s4[u].y, e[u][1] - mxw[u]) * fa.y) +
                                    (ldexp_pos(s4[u].z, e[u][2] - mxw[u]) * fb.x + ldexp_pos(s4[u].w, e[u][3] - mxw[u]) * fb.y)
                              : 0.0;
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int u = 0; u < RB; ++u) v[u] += __shfl_xor_sync(0xffffffffu, v[u], o);
          if (lane == 0)
#pragma unroll
            for (int u = 0; u < RB; ++u) {
              const int lr = (r0 + u) * ppr + et / lpp;
              if (lr < nrows) chunk[lr * cpp + cq / 32] = make_double2(v[u], (double)mxw[u]);
            }
        }
      };
      {
        const int rounds = (nrows + ppr - 1) / ppr;
        if (rounds <= 1) row_pass(std::integral_constant<int, 1>{});
        else row_pass(std::integral_constant<int, 4>{});
      }
      ebar();
      mark(1);
      // piece combine, one warp per row (rows ew, ew + 8, ...): lane k < cpp holds the warp partial k; exact
      // power-of-two rescaling to the piece maximum (REDUX), then a fixed shuffle tree over lanes 0..7
      for (int lr = ew; lr < nrows; lr += kResNE) {
        const double2 c = lane < cpp ? chunk[lr * cpp + lane] : make_double2(0.0, 0.0);
        const int mx = __reduce_max_sync(0xffffffffu, lane < cpp ? (int)c.y : INT_MIN);
        double r = lane < cpp ? c.x * pow2i((int)c.y - mx) : 0.0;
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
        if (h == 1) {
          if (lane == 0) {
            rowk[buf * MR + lr] = mx;
            rowr[buf * MR + lr] = r;
            rowf[buf * MR + lr] = alph[lr] * rcp_nomufu(r);
          }
        } else if (lane < h) {
          // (sum, shift) into cluster CTA `lane`'s slot [buf][lr][q] with st.async: the bytes complete the
          // transaction count of the receiver's barrier (no fence, no remote arrival)
          const unsigned ra = cluster_map(smem_u32(&rx[((size_t)buf * MR + lr) * h + q]), (unsigned)lane);
          const unsigned rb = cluster_map(smem_u32(rbar), (unsigned)lane);
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(ra),
                       "l"((unsigned long long)__double_as_longlong(r)), "r"(rb)
                       : "memory");
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(ra + 8u),
                       "l"((unsigned long long)__double_as_longlong((double)mx)), "r"(rb)
                       : "memory");
        }
      }
      if (h > 1) {
        mbar_wait(rbar, (uint32_t)t & 1u);
        for (int lr = ew; lr < nrows; lr += kResNE) {   // every CTA of the cluster combines the pieces in the same order
          const double2 c = lane < h ? rx[((size_t)buf * MR + lr) * h + lane] : make_double2(0.0, 0.0);
          const int mx = __reduce_max_sync(0xffffffffu, lane < h ? (int)c.y : INT_MIN);
          double r = lane < h ? c.x * pow2i((int)c.y - mx) : 0.0;
#pragma unroll
          for (int o = 2; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
          if (lane == 0) {
            rowk[buf * MR + lr] = mx;
            rowr[buf * MR + lr] = r;
            rowf[buf * MR + lr] = alph[lr] * rcp_nomufu(r);
          }
        }
      }
      ebar();
      mark(2);
      // ---- column pass: P_j = sum_i (alpha_i / r_i) t_ij over the CTA's rows, fixed point, one reduction each
      unsigned long long* dst = lsum + (size_t)sT * m + col0;
      for (int cq = et; cq < W4; cq += kResET) {
        const int4 k4 = reinterpret_cast<const int4*>(zk)[cq];
        const double2 fa = reinterpret_cast<const double2*>(zf)[2 * cq];
        const double2 fb = reinterpret_cast<const double2*>(zf)[2 * cq + 1];
        double P0 = 0.0, P1 = 0.0, P2 = 0.0, P3 = 0.0;
        for (int lr = 0; lr < nrows; ++lr) {
          const int Q = lr * W4 + cq;
          const float4 s4 = sb[Q];
          const int4 a4 = ash[Q];
          const int kM = rowk[buf * MR + lr];
          const double f = rowf[buf * MR + lr];
          P0 = fma(f, ldexp_pos(s4.x, k4.x - a4.x - kM) * fa.x, P0);
          P1 = fma(f, ldexp_pos(s4.y, k4.y - a4.y - kM) * fa.y, P1);
          P2 = fma(f, ldexp_pos(s4.z, k4.z - a4.z - kM) * fb.x, P2);
          P3 = fma(f, ldexp_pos(s4.w, k4.w - a4.w - kM) * fb.y, P3);
        }
        ulonglong2* cb2 = reinterpret_cast<ulonglong2*>(colbuf + 4 * cq);
        // multi-GPU: every partial carries 1 in the top byte (the rank-local sums count their contributions)
        const unsigned long long one = fused ? kCntOne : 0ull;
        cb2[0] = make_ulonglong2(one | (P0 > 0.0 ? __double2ull_rz(P0 * scale) : 0ull),
                                 one | (P1 > 0.0 ? __double2ull_rz(P1 * scale) : 0ull));
        cb2[1] = make_ulonglong2(one | (P2 > 0.0 ? __double2ull_rz(P2 * scale) : 0ull),
                                 one | (P3 > 0.0 ? __double2ull_rz(P3 * scale) : 0ull));
      }
      ebar();
      mark(3);
      // ---- device-wide step: the W partials are added into the iteration's column sums with coalesced 64-bit
      // integer reductions (red.global.add.u64: exact, so the order in which CTAs arrive does not matter); one
      // thread then releases the CTA's arrival on the group's cumulative counter and waits for the group's
      // ncl arrivals [multi-GPU: each CTA pushes its 1/ncl slice of the group's rank-local sums to every rank and
      // the ranks' pushes are counted the same way].
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = et + k * kResET;
        if (j < W) red_add_gpu(dst + j, colbuf[j]);
      }
      if (!fused) ebar();
      if (et == 0) {
        mbar_arrive(sgo);   // the k-sum warps compute the next iteration's s' while this one is reduced
        mbar_arrive(&sempty[buf]);
        if (fused) {   // (the counter is kept in step for a later unsharded launch on this workspace; no wait)
          asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p.lcnt + q) : "memory");
        } else {
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p.lcnt + q) : "memory");
          if (!wait_count(p.lcnt + q, (unsigned)p.ncl * (unsigned)(T + 1ull))) ctl[RCTL_TIMEOUT] = 1u;
        }
      }
      if (!fused) ebar();
      mark(4);
      // [multi-GPU] push this CTA's 1/ncl slice of the group's rank-local sums into every rank's exchange sums
      // with system-scope reductions; each pushed value carries 1 in its top byte, so a rank's exchange sum of a
      // column is complete when its count is nranks: no counter, no fence between the pushes and the readers
      if (fused) {
        // this thread's zeroing of its slice (previous iteration) precedes its pushes for every observer
        if (js0 + et < js1) {
          if (nr > 1) asm volatile("fence.acq_rel.sys;" ::: "memory");
          else asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        for (int jj = js0 + et; jj < js1; jj += kResET) {
          const int j = col0 + jj;
          unsigned long long v;   // the group's rank-local sum of the column, complete when its count is ncl
          if (!poll_sum1(lsum + (size_t)sT * m + j, (unsigned)p.ncl, v)) {
            timeout = true;
            break;
          }
          v = (v & kValMask) | kCntOne;
          for (int r = 0; r < nr; ++r) {   // the own rank's copy at GPU scope, the peers' at system scope
            if (r == p.rank) red_add_gpu(p.xsum[r] + (size_t)sX * m + j, v);
            else red_add_sys(p.xsum[r] + (size_t)sX * m + j, v);
          }
          // the pusher is the only reader of this rank-local sum: zero it now (the slot is reused three iterations
          // on, by CTAs that observed this thread's later pushes; the fence before those orders this store)
          st_relaxed_sys(lsum + (size_t)sT * m + j, 0ull);
        }
      }
      if (ctl[RCTL_TIMEOUT]) timeout = true;
      const unsigned long long* src = fused ? xown + (size_t)sX * m : lsum + (size_t)sT * m;
      // ---- q-update of the own columns: z_j += log beta_j - log c_j (every CTA of the group, same bits)
      // in split form, multiplicatively: 2^{kz_j} Fz_j <- 2^{kz_j} Fz_j beta_j / c_j, renormalised by exponent bits
      // (no log / exp per column); the thread's <= 4 columns are polled together until complete
      if (!timeout) {
        unsigned long long v[4];
        if (fused) {
          timeout |= !poll_sums4(src + col0, et, W, (unsigned)nr, v);
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (et + k * kResET < W) v[k] = ld_relaxed_sys(src + col0 + et + k * kResET);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int j = et + k * kResET;
          if (j < W && !timeout) {
            const double cj = (double)(v[k] & kValMask) * iscale;
            if (!(cj >= 1e-28)) underflow = true;
            int kz = zk[j];
            zf[j] = renorm_pow2(zf[j] * (bet[j] * rcp_nomufu(cj)), kz);
            zk[j] = kz;
          }
        }
      }
      // ---- zero this CTA's slice of the previous slot (read by every CTA before its reduction of this iteration)
      for (int j = js0 + et; j < js1; j += kResET) {
        if (fused) st_relaxed_sys(xown + (size_t)sXp * m + col0 + j, 0ull);   // (rank-local slots: at the push)
        else st_relaxed_sys(lsum + (size_t)sTp * m + col0 + j, 0ull);
      }
      timeout = bar_or(timeout);
      mark(5);
      st.iters = iters0 + t + 1;
      done = t + 1;
      // ---- monitor n sum_j |c_j - beta_j| from all m sums, fixed order: same value everywhere
      const bool need = (p.tol > 0.0 && st.iters % p.check_every == 0) || t == p.iters - 1;
      if (need && !timeout) {
        if (et == 0 && !fused)   // every column group's sums of this iteration are complete
          for (int g = 0; g < h; ++g)
            if (!wait_count(p.lcnt + g, (unsigned)p.ncl * (unsigned)(T + 1ull))) ctl[RCTL_TIMEOUT] = 1u;
        ebar();
        double dev = 0.0;
        {
          unsigned long long v[4];
          if (fused) {
            timeout |= !poll_sums4(src, et, m, (unsigned)nr, v);
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (et + k * kResET < m) v[k] = ld_relaxed_sys(src + et + k * kResET);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (et + k * kResET < m && !timeout) dev += fabs((double)(v[k] & kValMask) * iscale - p.beta[et + k * kResET]);
        }
        dev = warp_sum(dev);
        if (lane == 0) red[8 + ew] = dev;
        if (ctl[RCTL_TIMEOUT]) timeout = true;
        timeout = bar_or(timeout);
        st.residual = (((red[8] + red[9]) + (red[10] + red[11])) + ((red[12] + red[13]) + (red[14] + red[15]))) * (double)n;
        if (p.tol > 0.0 && st.iters % p.check_every == 0 && st.residual <= p.tol) {
          st.active = 0;
          st.converged = 1;
          halted = true;
        }
      }
      mark(6);
      if (timeout) halted = true;
      if (halted) break;
    }
    if (p.trace && et == 0)
      for (int k = 0; k < 7; ++k) p.trace[(size_t)blockIdx.x * 16 + 2 + k] = tr[k];
    if (halted && et == 0) *(volatile unsigned*)&ctl[RCTL_HALT] = 1u;
    if (halted && timeout && h > 1) {
      // A device-wide wait of this CTA gave up (a peer never arrived) while a cluster peer may have got past it
      // and now waits, with no time-out, for this CTA's row pieces of the next iteration: send it empty pieces so
      // that it reaches its own device-wide wait, times out there too and halts (no hang). Never on the fast path.
      const int bn = done & 1;
      for (int lr = ew; lr < nrows; lr += kResNE)
        if (lane < h) {
          const unsigned ra = cluster_map(smem_u32(&rx[((size_t)bn * MR + lr) * h + q]), (unsigned)lane);
          const unsigned rb = cluster_map(smem_u32(rbar), (unsigned)lane);
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(ra), "l"(0ull),
                       "r"(rb)
                       : "memory");
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(ra + 8u),
                       "l"(0ull), "r"(rb)
                       : "memory");
        }
    }
    ebar();
    // ---- outputs: z of the own columns (cluster 0's CTAs), w_hat of the own rows (piece 0's CTAs), state
    if (active0 && done > 0) {
      if (c == 0)
        for (int j = et; j < W; j += kResET) p.z_hat[col0 + j] = (double)zk[j] * COT_LN2 + log(zf[j]);
      const int fb = (done - 1) & 1;
      if (q == 0)
        for (int lr = et; lr < nrows; lr += kResET)
          p.w_hat[p.row_begin + lr0 + lr] = lal[lr] - ((double)rowk[fb * MR + lr] * COT_LN2 + log(rowr[fb * MR + lr]));
      if (b == 0 && et == 0) {
        SolverState out = p.state[0];
        out.iters = st.iters;
        out.residual = st.residual;
        out.active = st.active;
        out.converged = st.converged;
        p.state[0] = out;
        *reinterpret_cast<volatile unsigned long long*>(p.lcnt + 8) = Er + (unsigned long long)done;
        if (fused) *reinterpret_cast<volatile unsigned long long*>(p.xcnt[p.rank] + 8) = Ex + (unsigned long long)done;
      }
    }
    if (underflow) atomicOr(&p.state[0].flags, (int)STATE_UNDERFLOW);
    if (timeout) atomicOr(&p.state[0].flags, (int)STATE_PEER_TIMEOUT);
  }
  __syncthreads();
  if (h > 1) cluster_sync_all();   // no CTA leaves while a peer may still write its shared memory
}

__global__ void __launch_bounds__(kResThreads, 1) k_iter_res(const ResParams p) { res_body(p, blockIdx.x); }
__global__ void __launch_bounds__(kResThreads, 1) k_iter_res_emu(const __grid_constant__ ResMulti pm) {
  int v = 0;
  while (v + 1 < pm.nv && (int)blockIdx.x >= pm.base[v + 1]) ++v;
  res_body(pm.rp[v], (int)blockIdx.x - pm.base[v]);
}

// ------------------------------------------------------------------------------------------------- host
namespace {
int max_active_clusters(int h) {
  static std::mutex mu;
  static int cache[5] = {0, 0, 0, 0, 0};
  std::lock_guard<std::mutex> lk(mu);
  if (cache[h]) return cache[h];
  cudaFuncSetAttribute((void*)k_iter_res, cudaFuncAttributeMaxDynamicSharedMemorySize, kResMaxSmem);
  cudaFuncSetAttribute((void*)k_iter_res, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = h;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(h * 64);
  cfg.blockDim = dim3(kResThreads);
  cfg.dynamicSmemBytes = 200 * 1024;   // one CTA per SM whatever the layout
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nact = 0;
  if (cudaOccupancyMaxActiveClusters(&nact, (void*)k_iter_res, &cfg) != cudaSuccess) {
    cudaGetLastError();
    nact = 0;
  }
  cache[h] = nact > 0 ? nact : -1;
  return cache[h];
}
}  // namespace

// Configuration of the resident kernel for a rank holding R rows (Rlo: the smallest row count of any rank of
// the partition: the cluster count must be the same on every rank) with `sms` SMs. False if it does not fit.
bool res_config(int64_t n, int64_t m, int64_t R, int64_t Rlo, int sms, int nranks_emulated, ResCfg* out) {
  if (const char* ev = getenv("COT_RES"))
    if (atoi(ev) == 0) return false;
  int force_h = 0;
  if (const char* ev = getenv("COT_RES_H")) force_h = atoi(ev);
  bool found = false;
  ResCfg best{};
  double best_cost = 0.0;
  for (int h : {1, 2, 4}) {
    if (force_h && h != force_h) continue;
    if (m > 1024 || m % h != 0 || (m / h) % 128 != 0) continue;
    const int W = (int)(m / h);
    int ncl = sms / h;
    if (h > 1) {
      const int act = max_active_clusters(h);
      if (act <= 0) continue;
      ncl = std::min(ncl, act / std::max(1, nranks_emulated));
    }
    ncl = (int)std::min<int64_t>(ncl, Rlo);
    if (ncl < 1) continue;
    const int MR0 = (int)((R + ncl - 1) / ncl);
    const int MR = (MR0 + 1) & ~1;
    const int nq_max = MR0 * (W / 4);
    const int tq = (n % 4 == 0 && n <= 64) ? (int)(64 / n) : 0;   // 256 TMEM words per thread / 4n
    int nsq = std::max(0, nq_max - kResKT * tq);
    // shared memory left for quads; what does not fit is streamed from L2 every iteration -- allowed for up to a
    // quarter of the quads of a shard that stays L2-resident (the 4-GPU C4 shard: 512 quads, 66 streamed)
    const size_t fixed = res_layout((int)n, 0, nq_max, W, MR, h).total;
    const int cap = fixed >= (size_t)kResMaxSmem ? 0 : (int)(((size_t)kResMaxSmem - fixed) / ((size_t)16 * n));
    int nstream = 0;
    if (nsq > cap) {
      nstream = nsq - cap;
      nsq = cap;
    }
    const bool stream_ok = nstream == 0 || (nstream * 4 <= nq_max && (double)n * R * m * 4.0 <= 96e6 &&
                                            !(getenv("COT_RES_STREAM") && atoi(getenv("COT_RES_STREAM")) == 0));
    const ResLayout L = res_layout((int)n, nsq, nq_max, W, MR, h);
    if (getenv("COT_RES_DEBUG"))
      fprintf(stderr, "[res_config] n=%lld m=%lld R=%lld h=%d ncl=%d (active clusters %d) MR=%d quads=%d tq=%d nsq=%d "
              "streamed=%d smem=%zu%s\n",
              (long long)n, (long long)m, (long long)R, h, ncl, h > 1 ? max_active_clusters(h) : sms, MR0, nq_max, tq,
              nsq, nstream, L.total, (L.total > (size_t)kResMaxSmem || !stream_ok) ? " (does not fit)" : "");
    if (L.total > (size_t)kResMaxSmem || !stream_ok) continue;
    ResCfg c{h, W, ncl, MR, nq_max, tq, nsq, L.total};
    // fewest quads per CTA (the k-sum bound, a streamed quad counting double), scaled by the share of the SMs the
    // grid leaves idle (4-CTA clusters co-reside 33 at a time: 132 of 148 SMs); ties: the larger cluster while a
    // CTA holds few row pieces (fewer contributions per column sum), else the smaller one. Measured: the 8-way C4
    // shard 5.17 / 4.69 / 4.79 us per iteration at h = 1 / 2 / 4, the 4-way 9.65 (h = 2) / 9.73 (h = 4); C3 7
    // rows per CTA at h = 1 vs 14 at h = 2, whose longer column pass outweighs the cheaper reduction
    const double cost = (double)(nq_max + nstream) * (double)sms / (double)(ncl * h);
    if (!found || cost < best_cost * 0.999 || (cost <= best_cost * 1.001 && MR0 <= 8 && h > best.h)) {
      best_cost = cost;
      best = c;
      found = true;
    }
  }
  if (found && out) *out = best;
  return found;
}

bool res_eligible(const IterArgs& a, int sms) {
  if (a.B != 1 || a.dtype != COT_F32 || a.m % 4 != 0) return false;
  if (a.flags & (COT_DETERMINISTIC | COT_PRECOMPUTED | COT_FORCE_TMA | COT_FORCE_LDG | COT_DIAG_NO_COMPUTE |
                 COT_DIAG_NO_SYNC | COT_DIAG_NO_STREAM))
    return false;
  if (sms <= 0) sms = device_sm_count();
  return res_config(a.n, a.m, a.R, a.R, sms, 1, nullptr);
}

static void res_fill(const IterArgs& a, const Workspace& ws, const ResCfg& c, int iters, ResParams* p) {
  memset(p, 0, sizeof(*p));
  p->C = static_cast<const float*>(a.C);
  p->G = static_cast<const float*>(a.G);
  p->alpha = a.alpha;
  p->beta = a.beta;
  p->w_hat = a.w_hat;
  p->z_hat = a.z_hat;
  p->eps = a.eps;
  p->n = (int)a.n;
  p->m = (int)a.m;
  p->R = (int)a.R;
  p->row_begin = (int)a.row_begin;
  p->h = c.h;
  p->W = c.W;
  p->ncl = c.ncl;
  p->MR = c.MR;
  p->nq_max = c.nq_max;
  p->tq = c.tq;
  p->nsq = c.nsq;
  // throttle when the CTA's k-sums (one MUFU.EX2 per term, ~14 per clock) fit in the device-wide step (~6K clocks)
  p->throttle = (double)c.nq_max * 4.0 * (double)a.n / 14.0 < 6000.0 ? 1 : 0;
  if (const char* ev = getenv("COT_RES_THROTTLE")) p->throttle = atoi(ev) != 0;
  p->iters = iters;
  p->tol = a.tol;
  p->check_every = a.check_every > 0 ? a.check_every : 1;
  p->state = ws.state;
  p->lsum = ws.rsum;
  p->lcnt = ws.rcnt;
}

static unsigned long long* res_trace_buf() {
  static unsigned long long* buf = nullptr;
  if (!getenv("COT_TRACE")) return nullptr;
  if (!buf) cudaMalloc(&buf, 4096 * 16 * sizeof(unsigned long long));
  return buf;
}
static void res_trace_print(const unsigned long long* tb, int grid, int iters, cudaStream_t s) {
  std::vector<unsigned long long> hb((size_t)grid * 16);
  cudaStreamSynchronize(s);
  cudaMemcpy(hb.data(), tb, hb.size() * 8, cudaMemcpyDeviceToHost);
  const char* nm[9] = {"ksum_wait", "ksum_busy", "epi_wait_s", "row_pass", "row_xchg", "col_pass", "sync", "q_update",
                       "monitor"};
  fprintf(stderr, "[res trace] grid=%d iters=%d cycles/iter mean/max:", grid, iters);
  for (int k = 0; k < 9; ++k) {
    double a = 0, mx = 0;
    for (int b = 0; b < grid; ++b) {
      a += (double)hb[(size_t)b * 16 + k] / grid;
      mx = std::max(mx, (double)hb[(size_t)b * 16 + k]);
    }
    fprintf(stderr, " %s %.0f/%.0f", nm[k], a / std::max(1, iters), mx / std::max(1, iters));
  }
  fprintf(stderr, "\n");
}

static cudaError_t res_launch(void* fn, void* arg, int grid, int h, size_t smem, cudaStream_t s) {
  // one CTA per SM: each allocates all 512 TMEM columns, and CTAs spin on each other (two CTAs sharing an SM
  // would wait for each other's TMEM)
  smem = std::max<size_t>(smem, 120 * 1024);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (h > 1) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (h > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = h;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  attr[na].id = cudaLaunchAttributeCooperative;   // all CTAs co-resident (they wait on each other)
  attr[na].val.cooperative = 1;
  ++na;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kResThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = na;
  void* args[] = {arg};
  e = cudaLaunchKernelExC(&cfg, fn, args);
  if (e != cudaSuccess && h > 1) {
    // cooperative + cluster launch refused: the grid is sized to the co-resident cluster count, launch plainly
    cudaGetLastError();
    cfg.numAttrs = na - 1;
    e = cudaLaunchKernelExC(&cfg, fn, args);
  }
  return e;
}

cudaError_t launch_iter_res(const IterArgs& a, const Workspace& ws, int iters, cudaStream_t s) {
  ResCfg c;
  if (!res_config(a.n, a.m, a.R, a.R, device_sm_count(), 1, &c)) return cudaErrorInvalidConfiguration;
  if (!ws.rsum || !ws.rcnt) return cudaErrorInvalidValue;
  ResParams p;
  res_fill(a, ws, c, iters, &p);
  p.trace = res_trace_buf();
  if (p.trace) cudaMemsetAsync(p.trace, 0, 4096 * 16 * 8, s);
  cudaError_t e = res_launch((void*)k_iter_res, &p, c.h * c.ncl, c.h, c.smem, s);
  if (e == cudaSuccess && p.trace) res_trace_print(p.trace, c.h * c.ncl, iters, s);
  return e;
}

bool res_fused_config(const FusedRank& r, int nranks, bool emulate, ResCfg* c) {
  const IterArgs& a = r.a;
  if (a.B != 1 || a.dtype != COT_F32 || a.m % 4 != 0) return false;
  if (a.flags & (COT_DETERMINISTIC | COT_PRECOMPUTED | COT_FORCE_TMA | COT_FORCE_LDG | COT_DIAG_NO_COMPUTE |
                 COT_DIAG_NO_SYNC | COT_DIAG_NO_STREAM))
    return false;
  for (int q = 0; q < nranks; ++q)
    if (!r.xres[q]) return false;
  const int sms = emulate ? device_sm_count() / nranks : device_sm_count();
  const int64_t lo = a.m / nranks, hi = (a.m + nranks - 1) / nranks;
  const int64_t R = nranks == 1 ? a.R : hi, Rlo = nranks == 1 ? a.R : std::max<int64_t>(1, lo);
  return res_config(a.n, a.m, R, Rlo, sms, emulate ? nranks : 1, c);
}

cudaError_t launch_iter_res_fused(const FusedRank* r, int nv, int nranks, bool emulate, int iters, cudaStream_t s) {
  if (nv < 1 || nv > kMaxRanks || nranks < 1 || nranks > kMaxRanks || (emulate && nv != nranks) ||
      (!emulate && nv != 1))
    return cudaErrorInvalidValue;
  ResCfg c;
  if (!res_fused_config(r[0], nranks, emulate, &c)) return cudaErrorInvalidConfiguration;
  ResMulti pm;
  memset(&pm, 0, sizeof(pm));
  pm.nv = nv;
  pm.base[0] = 0;
  for (int v = 0; v < nv; ++v) {
    if (!r[v].ws.rsum || !r[v].ws.rcnt) return cudaErrorInvalidValue;
    if (r[v].a.R > (int64_t)c.ncl * ((c.nq_max / (c.W / 4)))) return cudaErrorInvalidConfiguration;
    ResParams& p = pm.rp[v];
    res_fill(r[v].a, r[v].ws, c, iters, &p);
    p.nranks = nranks;
    p.rank = r[v].rank;
    for (int q = 0; q < nranks; ++q) {
      p.xcnt[q] = reinterpret_cast<unsigned*>(r[v].xres[q]);
      p.xsum[q] = reinterpret_cast<unsigned long long*>(r[v].xres[q] + kXchgResHeader);
    }
    pm.base[v + 1] = pm.base[v] + c.h * c.ncl;
  }
  if (!emulate) {
    pm.rp[0].trace = res_trace_buf();
    if (pm.rp[0].trace) cudaMemsetAsync(pm.rp[0].trace, 0, 4096 * 16 * 8, s);
    cudaError_t e = res_launch((void*)k_iter_res, &pm.rp[0], pm.base[1], c.h, c.smem, s);
    if (e == cudaSuccess && pm.rp[0].trace) res_trace_print(pm.rp[0].trace, pm.base[1], iters, s);
    return e;
  }
  return res_launch((void*)k_iter_res_emu, &pm, pm.base[nv], c.h, c.smem, s);
}

int res_path_h(int64_t n, int64_t m, int64_t R) {
  ResCfg c;
  if (!res_config(n, m, R, R, device_sm_count(), 1, &c)) return 0;
  return c.h;
}

}  // namespace cot
