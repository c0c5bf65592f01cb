// K-BATCH-CHAIN: cluster-resident cyclic Sinkhorn for small problems (m <= 128: C5, C2) with the whole
// iteration chain of a problem inside ONE CTA. Same arithmetic as k_batch_cluster (k_batch_cluster.cu), organised
// around what the per-iteration dependency allows (Alg. 2 lines 4-5, log domain of eq. P:403-411):
//
//   s'_ij = sum_k exp2(a_ij - C_ijk log2e/eps)    does not depend on the iterate (a_ij = round(G_ij log2e/eps));
//   r_i   = sum_j s'_ij 2^{kz_j - a_ij - kM_i} Fz_j,   rho_i = alpha_i / r_i,
//   c_j   = sum_i rho_i t_ij,   z_hat_j += log beta_j - log c_j            (the chain: z -> r -> rho -> c -> z).
//
// One thread-block cluster of NCL CTAs per problem. CTAs 1..NCL-1 ("producers") hold rows of every cost block in
// shared memory (loaded once) and, every iteration, stream them and evaluate all n*m^2 Gibbs terms (FFMA +
// MUFU.EX2 + FADD) into s'_ij, which they store straight into the chain CTA's shared memory (DSMEM, double
// buffered: they run up to two iterations ahead) and signal with one remote mbarrier arrival per warp. CTA 0
// ("chain") holds s' of the whole m x m problem and runs the O(m^2) chain of every iteration alone: 16 warps,
// eight rows per warp, one float4 of columns per lane, the eight row sums by a transposed butterfly (18 shuffles
// instead of 80), rho broadcast back by shuffles, the column sums of the 16 warps' fp64 partials in a fixed tree,
// the q-update and the monitor -- no cluster barrier and no cross-SM hop on the per-iteration critical path (the
// k_batch_cluster chain has two cluster barriers and a DSMEM column pass per iteration). Bound: the producers'
// MUFU.EX2 (n*m^2 per problem per iteration on NCL-1 SMs); the chain CTA's SM runs no exponentials. For a batch
// that fits one wave (latency-bound, C2) and m = 128, two or four chain CTAs split the rows (a half or a quarter
// of the r-pass each) and exchange their parts of the column sums through DSMEM once per iteration (chain_role).
// Every sum has a fixed order (bitwise reproducible) and nothing is carried across launches but z_hat (the row
// shift kM_i is the exact per-row maximum every iteration), so launch boundaries do not change the iterates.
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

constexpr int kChainThreads = 512;
constexpr int kChainWarps = kChainThreads / 32;
constexpr int kChainRowsPerWarp = 8;        // m <= kChainWarps * 8 = 128
constexpr int kChainHeader = 128;           // barriers + stop flag at the start of every CTA's shared memory

struct ChainParams {
  const float* C;        // [B][n][m][m] (precomputed mode: S [B][1][m][m])
  const float* G;        // [B][m][m]
  const double* alpha;   // [B][m]
  const double* beta;    // [B][m]
  double* w_hat;         // [B][m]
  double* z_hat;         // [B][m]
  const double* eps;     // [B]
  SolverState* state;    // [B]
  double* zcache;        // [B][m][3]: z_hat as last written by this kernel, Fz, kz (exact split across launches)
  int n, m, ncl, RB;     // CTAs per cluster (nch chain CTAs + ncl - nch producers), rows per producer
  int nch;               // chain CTAs per cluster: 1, or 2 (m == 128: each holds half of the rows)
  int iters;
  double tol;
  long long check_every;
  int pre;
  int diag;              // diagnostics only (COT_CHAIN_DIAG=2): the chain skips its passes and hands every buffer
                         // straight back (timing of the producers and the DSMEM delivery alone; results invalid)
  unsigned long long* trace;   // diagnostics (COT_TRACE=1): [grid][8] cycle counters, or nullptr
};

__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// DSMEM store whose completion is counted on the destination CTA's mbarrier (complete_tx, release.cluster)
__device__ __forceinline__ void st_async_f4(uint32_t addr, float4 v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   addr),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(remote_bar)
               : "memory");
}
__device__ __forceinline__ void st_async_b64(uint32_t addr, unsigned long long v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(addr), "l"(v),
               "r"(remote_bar)
               : "memory");
}
__device__ __forceinline__ void st_cluster_release_u32(uint32_t addr, unsigned v) {
  asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// Remote arrival without a release fence (a release at cluster scope compiles to MEMBAR.ALL.GPU): used only to
// hand a buffer back to its writers after every read of it has completed (the values were consumed before a
// CTA barrier), so nothing needs ordering.
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar) : "memory");
}
// Phase test with CTA-scope acquire: the s' bytes land through st.async, counted by complete_tx on this CTA's own
// barrier, and the free signal carries no data; a cluster-scope acquire would add an L1 invalidation (CCTL.IVALL)
// after every successful test.
__device__ __forceinline__ bool mbar_test_cta(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Non-blocking phase test (same scope): issued early, its result is consumed later.
__device__ __forceinline__ bool mbar_probe_cta(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// f * 2^(eb - 896) for f = s'_ij in [2^-1/2, 1.42 n] (fp32) and a biased exponent eb = e + 896 with e <= 0 (the
// exact row shift makes every exponent <= 0), exactly, with e clamped below at -1000 (terms < 2^-999 come out
// ~1e-301: negligible); integer operations only. The bias (fp64 1023 - fp32 127) is carried in the column
// exponents kz_j + 896, so no per-element add is needed for it.
__device__ __forceinline__ double ldexp_biased(float f, int eb) {
  const unsigned bits = __float_as_uint(f);
  eb = max(eb, 896 - 1000);
  return __hiloint2double((int)((bits >> 3) + ((unsigned)eb << 20)), (int)(bits << 29));
}

// A chain CTA: every iteration of the problem on s' from the producers (FULL: m == 128, no masking). NCH = 1: the
// one chain CTA holds all m rows. NCH = 2 or 4 (FULL only; the latency-bound regime, C2): chain CTA c holds rows
// [c m/NCH, (c+1) m/NCH) -- 8/NCH rows per warp, 1/NCH of the r-pass -- and sends its part of the column sums to
// the other chain CTAs once per iteration through DSMEM (st.async + complete_tx on their barriers); all add the
// parts in the same order (((part 0 + part 1) + part 2) + part 3), so c_j, the q-update, the monitor and the stop
// decision are bitwise the same in every chain CTA.
template <bool FULL, int NCH>
__device__ __forceinline__ void chain_role(const ChainParams& p, const int64_t b, const int crank, unsigned char* smem,
                                           uint64_t* bars, float* sb, const float c2, const SolverState st0) {
  static_assert(NCH == 1 || ((NCH == 2 || NCH == 4) && FULL), "several chain CTAs need m == 128");
  constexpr int RPW = kChainRowsPerWarp / NCH;   // rows per warp
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = p.n, m = FULL ? 128 : p.m, mv = m >> 2, NP = p.ncl - NCH;   // FULL: compile-time offsets
  const int MH = m / NCH;                        // rows of this chain CTA: [row0, row0 + MH)
  const int row0 = crank * MH;
  const int wps = m + 2;   // warp-partial row stride: the column pass's four row groups fall in two bank halves
  unsigned* stopf = reinterpret_cast<unsigned*>(smem + 64);
  int* As = reinterpret_cast<int*>(sb + (size_t)2 * MH * m);           // [MH][m] a_ij
  double* wpart = reinterpret_cast<double*>(As + (size_t)MH * m);      // [16][m + 2] warp column partials
  double* zf = wpart + (size_t)kChainWarps * wps;                      // [m] Fz_j
  double* bcol = zf + m;                                               // [m] beta_j
  double* rstat = bcol + m;                                            // [MH][2] kM_i ln2, r_i
  double* red = rstat + 2 * MH;                                        // [32]
  int* zk = reinterpret_cast<int*>(red + 32);                          // [m] kz_j + 896 (biased: see ldexp_biased)
  double* xh = reinterpret_cast<double*>(zk + m);                      // NCH > 1: [2][NCH][m] column-sum parts
  for (int idx = threadIdx.x; idx < MH * m; idx += kChainThreads)
    As[idx] = __float2int_rn(__ldg(p.G + ((size_t)b * m + row0) * m + idx) * c2);
  // z_hat_j log2e = kz_j + log2 Fz_j: the split this kernel left in the workspace when z_hat still holds exactly
  // what it wrote (a launch continuing the previous one: no rounding at launch boundaries), else split afresh
  double* zc = p.zcache + (size_t)b * m * 3;
  for (int j = threadIdx.x; j < m; j += kChainThreads) {
    const double z = p.z_hat[b * m + j];
    const double cf = zc[3 * j + 1], ck = zc[3 * j + 2];
    // a cached split is used only if z_hat is bitwise what this kernel wrote and the entry is a split of it
    // (Fz in [2^-1/2, 2^1/2], kz within 1 of z log2e): stale or zeroed workspace memory never passes
    if (__double_as_longlong(z) == __double_as_longlong(zc[3 * j]) && cf >= 0.7071067811865475 &&
        cf <= 1.4142135623730951 && fabs(ck - rint(z * COT_LOG2E)) <= 1.0) {
      zf[j] = cf;
      zk[j] = (int)ck + 896;
    } else {
      int kz;
      zf[j] = split_z(z, kz);
      zk[j] = kz + 896;
    }
    bcol[j] = p.beta[b * m + j];
  }
  // after the transposed butterfly lane l holds the sum of the warp's row kk (RPW = 8: kk = 4 b4 + 2 b3 + b2,
  // RPW = 4: kk = 2 b4 + b3, RPW = 2: kk = b4, with bi the bits of l)
  const int kk = RPW == 8   ? ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1)
                 : RPW == 4 ? ((lane >> 4) & 1) * 2 + ((lane >> 3) & 1)
                            : ((lane >> 4) & 1);
  const int my_i = warp + kk * kChainWarps;   // local row
  const bool my_valid = FULL || my_i < m;
  const double my_alpha = my_valid ? p.alpha[b * m + row0 + my_i] : 0.0;
  const bool lane_ok = FULL || lane < mv;
  const int jc = lane_ok ? lane : 0;
  // NCH > 1: thread g < NCH - 1 of a column group sends this CTA's part of the column sums to chain CTA
  // (crank + 1 + g) % NCH: that CTA's copy of the parts, and its barrier
  const int gsend = threadIdx.x & 3;
  const uint32_t peer = (uint32_t)((crank + 1 + gsend) % NCH);
  const uint32_t xh_peer = NCH > 1 ? mapa_u32(smem_u32(xh), peer) : 0u;
  const uint32_t xbar_peer = NCH > 1 ? mapa_u32(smem_u32(&bars[5]), peer) : 0u;
  // a_ij of the thread's rows also in tensor memory (128 columns: four warps per 32-lane quarter, 32 columns each,
  // words 4k + v = a of row warp + 16k, column 4 jc + v): the r-pass reads them with LDTM (~12 cycles, a separate
  // datapath) instead of LDS.128 on this SM's busy shared-memory port
  unsigned* tslot = reinterpret_cast<unsigned*>(smem + 96);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned ta = *tslot + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)((warp >> 2) * 32);
#pragma unroll
  for (int k = 0; k < RPW; ++k) {
    const int i = warp + k * kChainWarps;
    const int ic = FULL || i < m ? i : 0;
    const int4 a4 = reinterpret_cast<const int4*>(As + (size_t)ic * m)[jc];
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ta + 4u * k), "r"(a4.x),
                 "r"(a4.y), "r"(a4.z), "r"(a4.w));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  SolverState st = st0;
  bool underflow = false;
  int t = 0;
  long long cw = 0, cr = 0, cc = 0;
  for (; t < p.iters; ++t) {
    const long long c0t = p.trace ? clock64() : 0;
    const int q = t & 1;
    const bool need = (p.tol > 0.0 && (st.iters + 1) % p.check_every == 0) || t == p.iters - 1;
    while (!mbar_test_cta(&bars[q], (uint32_t)((t >> 1) & 1))) {
    }
    // arm buffer q for iteration t + 2 (its phase of iteration t has completed; the producers fill it only after
    // the free signal below); NCH = 2: arm this iteration's column-half exchange (the peer's bytes may land
    // before the arming: the transaction count goes negative until then, and the phase cannot complete early
    // since the arrival is still pending)
    if (threadIdx.x == 0 && t + 2 < p.iters) mbar_arrive_expect_tx(&bars[q], (uint32_t)(MH * m * 4));
    if (NCH > 1 && threadIdx.x == 0) mbar_arrive_expect_tx(&bars[5 + q], (uint32_t)((NCH - 1) * m * 8));
    const long long c1t = p.trace ? clock64() : 0;
    if (p.diag & 2) {   // diagnostics: producers alone
      if (threadIdx.x < NP)
        mbar_arrive_cluster_relaxed(mapa_u32(smem_u32(&bars[2 + q]), (uint32_t)(threadIdx.x + NCH)));
      if (NCH > 1) {   // keep the exchange's phases moving: send zeros
        if (gsend < NCH - 1)
          st_async_b64(xh_peer + (uint32_t)(((q * NCH + crank) * m + (threadIdx.x >> 2)) * 8), 0ull,
                       xbar_peer + 8u * q);
        while (!mbar_test_cta(&bars[5 + q], (uint32_t)((t >> 1) & 1))) {
        }
      }
      st.iters += 1;
      continue;
    }
    // ---- r-pass: the warp's RPW rows, one float4 of columns per lane:
    //      u_ij = s'_ij 2^{kz_j - a_ij - kM_i},  r_i = sum_j u_ij Fz_j,  P_j = Fz_j sum_i rho_i u_ij
    const int4 k4 = reinterpret_cast<const int4*>(zk)[jc];
    const double2 fa = reinterpret_cast<const double2*>(zf)[2 * jc];
    const double2 fb = reinterpret_cast<const double2*>(zf)[2 * jc + 1];
    const double fz[4] = {fa.x, fa.y, fb.x, fb.y};
    const float* sq = sb + (size_t)q * MH * m;
    double uu[RPW][4], ls[RPW];
    int kM[RPW];
#pragma unroll
    for (int k = 0; k < RPW; ++k) {
      const int i = warp + k * kChainWarps;
      const bool ok = FULL || (i < m && lane < mv);
      const int ic = FULL || i < m ? i : 0;
      const float4 s4 = reinterpret_cast<const float4*>(sq + (size_t)ic * m)[jc];
      int4 a4;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(a4.x), "=r"(a4.y), "=r"(a4.z), "=r"(a4.w)
                   : "r"(ta + 4u * k));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      (void)ic;
      const int ex[4] = {k4.x - a4.x, k4.y - a4.y, k4.z - a4.z, k4.w - a4.w};   // kz_j + 896 - a_ij
      const int em = max(max(ex[0], ex[1]), max(ex[2], ex[3]));
      // exact row shift kM_i = max_j (kz_j - a_ij): the largest term is >= 1/2
      kM[k] = __reduce_max_sync(0xffffffffu, ok ? em : -0x7fffffff) - 896;
      const float sv[4] = {s4.x, s4.y, s4.z, s4.w};
      ls[k] = 0.0;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        uu[k][v] = ldexp_biased(sv[v], ex[v] - kM[k]);
        if (!FULL && !ok) uu[k][v] = 0.0;
        ls[k] = fma(uu[k][v], fz[v], ls[k]);
      }
    }
    // the RPW row sums by a transposed butterfly: each level keeps half of the rows and sends the other half
    const bool h4 = lane & 16, h3 = lane & 8, h2 = lane & 4;
    double r;
    if constexpr (RPW == 8) {
      double a4s[4], a2s[2];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        a4s[k] = (h4 ? ls[k + 4] : ls[k]) + __shfl_xor_sync(0xffffffffu, h4 ? ls[k] : ls[k + 4], 16);
#pragma unroll
      for (int k = 0; k < 2; ++k)
        a2s[k] = (h3 ? a4s[k + 2] : a4s[k]) + __shfl_xor_sync(0xffffffffu, h3 ? a4s[k] : a4s[k + 2], 8);
      r = (h2 ? a2s[1] : a2s[0]) + __shfl_xor_sync(0xffffffffu, h2 ? a2s[0] : a2s[1], 4);
    } else if constexpr (RPW == 4) {
      double a2s[2];
#pragma unroll
      for (int k = 0; k < 2; ++k)
        a2s[k] = (h4 ? ls[k + 2] : ls[k]) + __shfl_xor_sync(0xffffffffu, h4 ? ls[k] : ls[k + 2], 16);
      r = (h3 ? a2s[1] : a2s[0]) + __shfl_xor_sync(0xffffffffu, h3 ? a2s[0] : a2s[1], 8);
      r += __shfl_xor_sync(0xffffffffu, r, 4);
    } else {
      r = (h4 ? ls[1] : ls[0]) + __shfl_xor_sync(0xffffffffu, h4 ? ls[0] : ls[1], 16);
      r += __shfl_xor_sync(0xffffffffu, r, 8);
      r += __shfl_xor_sync(0xffffffffu, r, 4);
    }
    r += __shfl_xor_sync(0xffffffffu, r, 2);
    r += __shfl_xor_sync(0xffffffffu, r, 1);
    const double rho_my = my_valid ? my_alpha * __drcp_rn(r) : 0.0;   // alpha_i / r_i (this SM's MUFU is idle)
    if (need && (lane & (32 / RPW - 1)) == 0 && my_valid) {   // the row statistics of w_hat (last iteration)
      int km = 0;
#pragma unroll
      for (int k = 0; k < RPW; ++k) km = k == kk ? kM[k] : km;
      rstat[2 * my_i] = (double)km * COT_LN2;
      rstat[2 * my_i + 1] = r;
    }
    double P[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < RPW; ++k) {   // rows in order
      const int src = RPW == 8   ? ((k >> 2) & 1) * 16 + ((k >> 1) & 1) * 8 + (k & 1) * 4
                      : RPW == 4 ? ((k >> 1) & 1) * 16 + (k & 1) * 8
                                 : k * 16;
      const double rho = __shfl_sync(0xffffffffu, rho_my, src);
#pragma unroll
      for (int v = 0; v < 4; ++v) P[v] = fma(rho, uu[k][v], P[v]);
    }
    if (lane_ok) {
      double2* wp = reinterpret_cast<double2*>(wpart + (size_t)warp * wps);
      wp[2 * lane] = make_double2(P[0] * fz[0], P[1] * fz[1]);
      wp[2 * lane + 1] = make_double2(P[2] * fz[2], P[3] * fz[3]);
    }
    __syncthreads();
    const long long c2t = p.trace ? clock64() : 0;
    // s' buffer q has been read: the producers may fill it with iteration t + 2
    if (threadIdx.x < NP)
      mbar_arrive_cluster_relaxed(mapa_u32(smem_u32(&bars[2 + q]), (uint32_t)(threadIdx.x + NCH)));
    // ---- column pass: 4 threads per column (4 warps' partials each, then a fixed xor tree) and the q-update
    //      z_hat_j += log beta_j - log c_j carried on the split: Fz_j beta_j / c_j = M 2^E, M in [2^-1/2, 2^1/2)
    //      -> kz_j += E, Fz_j = M (no log, no exp on the critical path)
    const int col = threadIdx.x >> 2, g = threadIdx.x & 3;
    const bool cok = FULL || col < m;
    double c = 0.0;
    if (cok) {
      const double* wp = wpart + (size_t)(4 * g) * wps + col;
      c = (wp[0] + wp[wps]) + (wp[2 * (size_t)wps] + wp[3 * (size_t)wps]);
    }
    c += __shfl_xor_sync(0xffffffffu, c, 1);   // (a0 + a1) + (a2 + a3) in every lane of the group: the
    c += __shfl_xor_sync(0xffffffffu, c, 2);   // additions commute bitwise
    if constexpr (NCH > 1) {   // swap the parts: c_j = ((part 0 + part 1) + part 2) + part 3 in every chain CTA
      double* xq = xh + (size_t)q * NCH * m;
      if (g == 0) xq[crank * m + col] = c;
      if (g < NCH - 1)
        st_async_b64(xh_peer + (uint32_t)(((q * NCH + crank) * m + col) * 8),
                     (unsigned long long)__double_as_longlong(c), xbar_peer + 8u * q);
      while (!mbar_test_cta(&bars[5 + q], (uint32_t)((t >> 1) & 1))) {
      }
      if (g == 0) {
        c = xq[col];
#pragma unroll
        for (int h = 1; h < NCH; ++h) c += xq[h * m + col];
      }
    }
    double dev = 0.0;
    if (cok && g == 0) {
      const double bj = bcol[col];
      dev = fabs(c - bj);
      underflow |= !(c >= 1e-28);
      const double R = (zf[col] * bj) * __drcp_rn(c);
      const int hi = __double2hiint(R);
      int E = (hi >> 20) - 1023;
      double M = __hiloint2double((hi & 0x000FFFFF) | 0x3FF00000, __double2loint(R));   // [1, 2)
      if (M > 1.4142135623730951) {
        M *= 0.5;
        E += 1;
      }
      zf[col] = M;
      zk[col] += E;
    }
    if (need) {
      dev = warp_sum(dev);
      if (lane == 0) red[warp] = dev;
    }
    __syncthreads();
    if (p.trace) {
      const long long c3t = clock64();
      cw += c1t - c0t;
      cr += c2t - c1t;
      cc += c3t - c2t;
    }
    st.iters += 1;
    if (need) {
      double d = 0.0;
#pragma unroll
      for (int w = 0; w < kChainWarps; ++w) d += red[w];
      st.residual = d * (double)n;
    }
    if (p.tol > 0.0 && st.iters % p.check_every == 0 && st.residual <= p.tol) {
      st.active = 0;
      st.converged = 1;
      ++t;
      break;
    }
  }
  if (p.trace && threadIdx.x == 0 && b < 64) {
    unsigned long long* tp = p.trace + (size_t)blockIdx.x * 8;
    tp[0] = cw;
    tp[1] = cr;
    tp[2] = cc;
  }
  // stop the producers (they may be up to two iterations ahead, waiting for a buffer); with several chain CTAs
  // all stop at the same iteration (identical decisions) and CTA 0 signals
  if (crank == 0 && threadIdx.x < NP)
    st_cluster_release_u32(mapa_u32(smem_u32(stopf), (uint32_t)(threadIdx.x + NCH)), 1u);
  for (int i = threadIdx.x; i < MH; i += kChainThreads)
    if (t > 0) {
      const int64_t gi = b * m + row0 + i;
      p.w_hat[gi] = log(p.alpha[gi]) - rstat[2 * i] - log(rstat[2 * i + 1]);
    }
  if (crank == 0)
    for (int j = threadIdx.x; j < m; j += kChainThreads) {   // z_hat_j = (kz_j + log2 Fz_j) ln 2, and its split
      const int kz = zk[j] - 896;
      const double z = (double)kz * COT_LN2 + log(zf[j]);
      p.z_hat[b * m + j] = z;
      zc[3 * j] = z;
      zc[3 * j + 1] = zf[j];
      zc[3 * j + 2] = (double)kz;
    }
  if (underflow) atomicOr(&p.state[b].flags, (int)STATE_UNDERFLOW);
  if (crank == 0 && threadIdx.x == 0) {
    SolverState out = p.state[b];
    out.iters = st.iters;
    out.residual = st.residual;
    out.active = st.active;
    out.converged = st.converged;
    p.state[b] = out;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(*tslot));
}

__global__ void __launch_bounds__(kChainThreads, 1) k_batch_chain(const __grid_constant__ ChainParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const int ncl = p.ncl;
  const int64_t b = blockIdx.x / ncl;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = p.n, m = p.m, mv = m >> 2;
  // header: [0] [1] chain: s' buffer q full (one arrival -- the chain's own expect_tx of its rows' bytes -- and the
  // producers' st.async transaction bytes per phase); [2] [3] producer: s' buffer q free (one arrival by each chain
  // CTA per phase); [4] producer: cost rows loaded; [5] [6] chain (nch > 1): the other chain CTAs' parts of the
  // column sums of iteration parity q arrived; stop flag at byte 64
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  unsigned* stopf = reinterpret_cast<unsigned*>(smem + 64);
  float* sbuf = reinterpret_cast<float*>(smem + kChainHeader);   // chain: [2][m][m] s'; producer: C rows

  const SolverState st0 = p.state[b];
  if (!st0.active) return;                                        // cluster-uniform
  const double inv_eps = 1.0 / p.eps[b];
  const float c2 = (float)(COT_LOG2E * inv_eps);
  const int nch = p.nch;
  if (threadIdx.x == 0) {
    if (crank < nch) {
      const uint32_t bytes = (uint32_t)(m / nch * m * 4);
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      mbar_init(&bars[5], 1);
      mbar_init(&bars[6], 1);
      // arm the buffers of iterations 0 and 1 (an armed phase that never receives data is never waited on)
      if (p.iters > 0) mbar_arrive_expect_tx(&bars[0], bytes);
      if (p.iters > 1) mbar_arrive_expect_tx(&bars[1], bytes);
    } else {
      mbar_init(&bars[2], (uint32_t)nch);
      mbar_init(&bars[3], (uint32_t)nch);
      mbar_init(&bars[4], 1);
    }
    *stopf = 0u;
    fence_mbar_init();
  }
  cluster.sync();

  if (crank >= nch) {
    // ============================================================================ producer
    const int i0 = (crank - nch) * p.RB;
    const int nrows = max(0, min(p.RB, m - i0));
    float* Cs = sbuf;                                             // [nrows][n][m]
    if (threadIdx.x == 0 && nrows > 0) {
      const uint32_t row_bytes = (uint32_t)m * 4u;
      mbar_arrive_expect_tx(&bars[4], (uint32_t)nrows * (uint32_t)n * row_bytes);
      const uint64_t pol = policy_evict_first();
      for (int i = 0; i < nrows; ++i)
        for (int k = 0; k < n; ++k)
          bulk_g2s(Cs + ((size_t)i * n + k) * m, p.C + (((size_t)b * n + k) * m + i0 + i) * m, row_bytes, &bars[4],
                   pol);
    }
    // the warp's rows (w, w + 16): integer shifts a_ij straight from G (as float, the k-sum's FFMA operand)
    float gcr[2][4], pf[2][4];
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int i = warp + rr * kChainWarps;
      const float4 g4 = (i < nrows && lane < mv)
                            ? __ldg(reinterpret_cast<const float4*>(p.G + ((size_t)b * m + i0 + i) * m) + lane)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
      const float gv[4] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        gcr[rr][v] = (float)__float2int_rn(gv[v] * c2);
        // precomputed mode (NEXT-1): the G-shifted S_ij rescaled to the same convention, S_ij 2^{a_ij - G_ij c2}
        pf[rr][v] = p.pre ? ex2(fmaf(-gv[v], c2, gcr[rr][v])) : 1.f;
      }
    }
    if (nrows > 0) mbar_wait(&bars[4], 0);
    // destination of each of the warp's rows: the chain CTA holding it (chain CTA c holds rows [c m/nch,
    // (c+1) m/nch)), its local row there, that CTA's s' buffers and full barriers
    const int mh = m / nch;
    uint32_t rs_buf[2], rfull[2];
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int gi = i0 + warp + rr * kChainWarps;
      const int dc = min(gi / mh, nch - 1);
      rs_buf[rr] = mapa_u32(smem_u32(sbuf), (uint32_t)dc) + (uint32_t)((gi - dc * mh) * m * 4);
      rfull[rr] = mapa_u32(smem_u32(&bars[0]), (uint32_t)dc);
    }
    long long tk = 0, tw = 0, tsv = 0;
    for (int t = 0; t < p.iters; ++t) {
      const long long c0t = p.trace ? clock64() : 0;
      // buffer q is free once the chain has finished the r-pass of iteration t - 2 (no wait for the first two);
      // it almost always is by now: probe before the k-sum, so that the probe's trip through the SM's
      // shared-memory pipe (queued behind the other warps' MUFU.EX2) overlaps the k-sum
      const int q = t & 1;
      const uint32_t par = (uint32_t)(((t >> 1) - 1) & 1);
      bool freed = t < 2 || mbar_probe_cta(&bars[2 + q], par);
      float s[2][4];
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
#pragma unroll
        for (int v = 0; v < 4; ++v) s[rr][v] = 0.f;
        const int i = warp + rr * kChainWarps;
        if (i >= nrows || lane >= mv) continue;
        const float4* crow = reinterpret_cast<const float4*>(Cs + (size_t)i * n * m);
        if (p.pre) {
          const float4 c = crow[lane];
          s[rr][0] = c.x * pf[rr][0];
          s[rr][1] = c.y * pf[rr][1];
          s[rr][2] = c.z * pf[rr][2];
          s[rr][3] = c.w * pf[rr][3];
          continue;
        }
        int k = 0;
        // blocks of 4 k: 16 independent MUFU.EX2 issued back to back, summed in a fixed pairwise order
        for (; k + 4 <= n; k += 4) {
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
        for (; k < n; ++k) {
          const float4 c = crow[(size_t)k * mv + lane];
          s[rr][0] += ex2(fmaf(-c.x, c2, gcr[rr][0]));
          s[rr][1] += ex2(fmaf(-c.y, c2, gcr[rr][1]));
          s[rr][2] += ex2(fmaf(-c.z, c2, gcr[rr][2]));
          s[rr][3] += ex2(fmaf(-c.w, c2, gcr[rr][3]));
        }
      }
      const long long c1t = p.trace ? clock64() : 0;
      // else poll: the whole warp (one instruction, a uniform result, no shuffle)
      bool go = true;
      if (!freed) {
        while (!mbar_test_cta(&bars[2 + q], par)) {
          if (*(volatile unsigned*)stopf) {   // the chain has stopped (it converged, or its launch ends)
            go = false;
            break;
          }
        }
      }
      if (!go) break;
      const long long c2t = p.trace ? clock64() : 0;
      // fire and forget: each 16-byte store counts its bytes on the chain's full[q] barrier when it lands
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const int i = warp + rr * kChainWarps;
        if (i < nrows && lane < mv)
          st_async_f4(rs_buf[rr] + (uint32_t)(((size_t)q * mh * m + 4 * lane) * 4),
                      make_float4(s[rr][0], s[rr][1], s[rr][2], s[rr][3]), rfull[rr] + 8u * (uint32_t)q);
      }
      if (p.trace) {
        const long long c3t = clock64();
        tk += c1t - c0t;
        tw += c2t - c1t;
        tsv += c3t - c2t;
      }
    }
    if (p.trace && threadIdx.x == 0 && b < 64) {
      unsigned long long* tp = p.trace + (size_t)blockIdx.x * 8;
      tp[0] = tk;
      tp[1] = tw;
      tp[2] = tsv;
    }
  } else {
    // ============================================================================ chain
    if (m == kChainWarps * kChainRowsPerWarp) {
      if (nch == 4)
        chain_role<true, 4>(p, b, crank, smem, bars, sbuf, c2, st0);
      else if (nch == 2)
        chain_role<true, 2>(p, b, crank, smem, bars, sbuf, c2, st0);
      else
        chain_role<true, 1>(p, b, crank, smem, bars, sbuf, c2, st0);
    } else {
      chain_role<false, 1>(p, b, crank, smem, bars, sbuf, c2, st0);
    }
  }
  cluster.sync();   // no CTA leaves while another may still write into its shared memory
}
// ------------------------------------------------------------------------------------------ launcher
namespace {
struct ChainCfg {
  int ncl, RB, nch;
  size_t smem;
};

// chain CTA: s' x 2 and a_ij of its mh rows, warp partials, Fz, beta, row stats, scratch, kz, column-sum parts
size_t chain_smem_chain(int64_t m, int nch) {
  const int64_t mh = m / nch;
  return kChainHeader + (size_t)2 * mh * m * 4 + (size_t)mh * m * 4 + (size_t)kChainWarps * (m + 2) * 8 +
         (size_t)m * 8 + (size_t)m * 8 + (size_t)mh * 16 + 32 * 8 + (size_t)m * 4 + (nch > 1 ? (size_t)2 * nch * m * 8 : 0);
}

bool chain_shape(int64_t n, int64_t m, int ncl, int nch, ChainCfg* c) {
  const int np = ncl - nch;
  if (np < 1 || m < 1) return false;
  if (nch > 1 && m != kChainWarps * kChainRowsPerWarp) return false;   // several chain CTAs: m == 128 only
  if (nch != 1 && nch != 2 && nch != 4) return false;
  const int RB = (int)((m + np - 1) / np);
  if (RB > 2 * kChainWarps) return false;   // two rows per producer warp
  const size_t prod = kChainHeader + (size_t)RB * n * m * 4;
  const size_t smem = std::max(prod, chain_smem_chain(m, nch));
  if (smem > 226 * 1024) return false;
  c->ncl = ncl;
  c->RB = RB;
  c->nch = nch;
  c->smem = smem;
  return true;
}

int chain_active_clusters(const ChainCfg& c) {
  // a few shapes per process (the launcher may probe two per call): cached, the occupancy query is not free;
  // calls on distinct streams may run concurrently (include/cyclicot.h)
  static std::mutex mu;
  static int64_t keys[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
  static int vals[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  static int next = 0;
  const int64_t key = (int64_t)c.smem * 32 + c.ncl;
  std::lock_guard<std::mutex> lock(mu);
  for (int i = 0; i < 8; ++i)
    if (keys[i] == key) return vals[i];
  cudaFuncSetAttribute((void*)k_batch_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem);
  if (c.ncl > 8) cudaFuncSetAttribute((void*)k_batch_chain, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(c.ncl * 64));
  cfg.blockDim = dim3(kChainThreads);
  cfg.dynamicSmemBytes = c.smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = c.ncl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nact = 0;
  if (cudaOccupancyMaxActiveClusters(&nact, (void*)k_batch_chain, &cfg) != cudaSuccess) {
    cudaGetLastError();
    nact = 0;
  }
  keys[next] = key;
  vals[next] = nact;
  next = (next + 1) & 7;
  return nact;
}

// Shape: 8-CTA clusters while the batch fits one wave of them (latency: C2) -- with two chain CTAs splitting the
// rows when m == 128 (6 producers), else one (7 producers) --, else 6-CTA clusters with one chain CTA (22
// co-resident vs 15: throughput, C5), else any feasible size. COT_CHAIN_NCL / COT_CHAIN_NCH force.
bool chain_config(int64_t n, int64_t m, int64_t B, ChainCfg* c) {
  const char* nchv = getenv("COT_CHAIN_NCH");
  const int nch_forced = nchv ? atoi(nchv) : 0;
  if (const char* ev = getenv("COT_CHAIN_NCL")) return chain_shape(n, m, atoi(ev), nch_forced ? nch_forced : 1, c);
  // one wave of 8-CTA clusters with as many chain CTAs as the producers' shared memory allows (4 producers x 32
  // rows, 6 x 22, 7 x 19). (16-CTA clusters, 4 chain CTAs + 12 producers, measured slower on C2: 1.79 vs 1.69 us
  // per iteration, the exchange between the chain CTAs takes longer; COT_CHAIN_NCL=16 still runs them.)
  ChainCfg c8;
  bool h8 = false;
  if (nch_forced)
    h8 = chain_shape(n, m, 8, nch_forced, &c8);
  else
    for (int nch : {4, 2, 1})
      if ((h8 = chain_shape(n, m, 8, nch, &c8))) break;
  if (h8 && B > 0 && B <= chain_active_clusters(c8)) {
    *c = c8;
    return true;
  }
  for (int ncl : {6, 7, 5, 8, 4, 3, 2})
    if (chain_shape(n, m, ncl, nch_forced ? nch_forced : 1, c) && (B <= 0 || chain_active_clusters(*c) > 0))
      return true;
  return false;
}
}  // namespace

bool batch_chain_eligible(const IterArgs& a) {
  if (a.dtype != COT_F32 || a.m % 4 != 0 || a.m > 128 || a.R != a.m ||
      (a.flags & (COT_FORCE_LDG | COT_FORCE_TMA)))
    return false;
  if (const char* ev = getenv("COT_BATCH_CHAIN"))
    if (atoi(ev) == 0) return false;
  ChainCfg c;
  return chain_config(a.n, a.m, 0, &c);
}

cudaError_t launch_batch_chain(const IterArgs& a, const Workspace& ws, int iters, cudaStream_t s) {
  ChainCfg cc;
  if (!chain_config(a.n, a.m, a.B, &cc)) return cudaErrorInvalidConfiguration;
  ChainParams p;
  p.C = static_cast<const float*>(a.C);
  p.G = static_cast<const float*>(a.G);
  p.alpha = a.alpha;
  p.beta = a.beta;
  p.w_hat = a.w_hat;
  p.z_hat = a.z_hat;
  p.eps = a.eps;
  p.state = ws.state;
  p.zcache = ws.zcache;
  p.n = (int)a.n;
  p.m = (int)a.m;
  p.ncl = cc.ncl;
  p.RB = cc.RB;
  p.nch = cc.nch;
  p.iters = iters;
  p.tol = a.tol;
  p.check_every = a.check_every > 0 ? a.check_every : 1;
  p.pre = (a.flags & COT_PRECOMPUTED) ? 1 : 0;
  p.diag = getenv("COT_CHAIN_DIAG") ? (atoi(getenv("COT_CHAIN_DIAG")) & 2) : 0;
  cudaError_t e = cudaFuncSetAttribute((void*)k_batch_chain, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)cc.smem);
  if (e == cudaSuccess && cc.ncl > 8)
    e = cudaFuncSetAttribute((void*)k_batch_chain, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.B * cc.ncl));
  cfg.blockDim = dim3(kChainThreads);
  cfg.dynamicSmemBytes = cc.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cc.ncl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static unsigned long long* trace_buf = nullptr;   // diagnostics only (COT_TRACE=1)
  p.trace = nullptr;
  if (getenv("COT_TRACE")) {
    if (!trace_buf) cudaMalloc(&trace_buf, 64 * 16 * 8 * sizeof(unsigned long long));
    cudaMemsetAsync(trace_buf, 0, 64 * 16 * 8 * sizeof(unsigned long long), s);
    p.trace = trace_buf;
  }
  void* args[] = {&p};
  e = cudaLaunchKernelExC(&cfg, (void*)k_batch_chain, args);
  if (e == cudaSuccess && p.trace) {
    const int nb = (int)std::min<int64_t>(a.B, 64);
    std::vector<unsigned long long> h((size_t)nb * cc.ncl * 8);
    cudaStreamSynchronize(s);
    cudaMemcpy(h.data(), p.trace, h.size() * 8, cudaMemcpyDeviceToHost);
    double ch[3] = {0, 0, 0}, pr[3] = {0, 0, 0};
    for (int c = 0; c < nb * cc.ncl; ++c)
      for (int k = 0; k < 3; ++k) {
        const double v = (double)h[(size_t)c * 8 + k] / std::max(iters, 1);
        if (c % cc.ncl < cc.nch) ch[k] += v / nb / cc.nch; else pr[k] += v / nb / (cc.ncl - cc.nch);
      }
    fprintf(stderr, "[cot chain trace] cluster %d (%d chain CTAs), %d problems traced; per-iter cycles: chain wait %.0f "
            "r-pass %.0f col-pass %.0f | producer k-sum %.0f wait-free %.0f store %.0f\n", cc.ncl, cc.nch, nb, ch[0], ch[1], ch[2],
            pr[0], pr[1], pr[2]);
  }
  return e;
}

}  // namespace cot
