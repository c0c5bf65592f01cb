// Internal host/device interface of libcyclicot: workspace layout, row-unit plan, kernel launchers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/cyclicot.h"

namespace cot {

// Per-problem solver state kept in the workspace (32 bytes).
struct SolverState {
  long long iters;   // iterations performed on this problem
  int active;        // 1 while iterating; 0 once converged (frozen)
  int converged;     // 1 if the monitor reached tol
  double residual;   // last monitor n*sum_j |c_j - beta_j| (after the p-update of the last iteration)
  int flags;         // bit 0: marginal validation failed; bit 1: column underflow
  int pad;
};
// STATE_DET_RANGE: set by cerot_init when sum(alpha) >= 2^7 (not an error by itself); a COT_DETERMINISTIC launch
// on such a problem refuses to iterate and sets STATE_DET_REFUSED (cerot_state: COT_E_ARG).
enum { STATE_BAD_MARGINAL = 1, STATE_UNDERFLOW = 2, STATE_PEER_TIMEOUT = 4, STATE_DET_RANGE = 8,
       STATE_DET_REFUSED = 16 };
constexpr double kDetAlphaMax = 128.0;   // 2^7: every fixed-point column partial stays below 2^8

constexpr int kMaxRanks = 8;   // fused multi-GPU exchange: ranks of one row partition (one 8-GPU node)
constexpr size_t kXchgHeader = 256;   // exchange buffer: epoch counter, then the LL lines
// ... then the region of K-ITER-RES's exchange: [8] arrival counters + epoch (u64), then [3][m] integer sums
constexpr size_t kXchgResHeader = 64;
size_t xchg_res_offset(int64_t m, int nranks);

// Rows of each problem are cut into units of `rpu` consecutive rows; units are the work items of the
// row kernels (K-ITER, K-PLAN) and each unit writes one fp64 column-partial row. `upp` units per
// problem, U = B * upp in total, processed by `grid` persistent CTAs (unit u -> CTA u % grid).
struct UnitPlan {
  int64_t rpu, upp, U;
  int grid;
};
UnitPlan unit_plan(int64_t B, int64_t R, int sm_count);

constexpr int kReportDoubles = 8;   // cot_report field order: objective .. residual
constexpr int kPlanScalars = 4;     // per unit: transport, entropy sum, row |r - alpha| sum, mass
constexpr int kPlanBufHead = 5;     // plan buffer: 4 scalars + sum_{held rows} w_hat_i alpha_i, then m column sums

struct Workspace {
  void* G;                 // [B][m][m] dtype
  int32_t* A;              // [B][m][m]
  double* partials[2];     // [U][m] x 2 (ping-pong by iteration parity)
  double* plan_scal;       // [U][kPlanScalars]
  double* resid_part;      // [B][ceil(m/32)]
  SolverState* state;      // [B]
  unsigned* counters;      // [B] last-block-done tickets (self-resetting)
  unsigned* grid_bar;      // [4] two device-wide barriers of the persistent TMA kernel (count, generation)
  unsigned* loopctl;       // [4] cerot_solve's device-side loop (CUDA graph while-node): iterations launched
  int32_t* nonfinite;      // [1]
  double* report;          // [B][kReportDoubles]
  double* c_local;         // [B][m] column sums over the held rows (sharded path)
  double* c_global;        // [B][m] column sums after the cross-GPU reduction
  double* plan_buf;        // [B][kPlanBufHead + m] local plan reductions (allreduced in place)
  double* rowscal;         // [B][m][4] per-row plan scalars of the C-SROT report
  double* zcache;          // [B][m][3] k_batch_chain: z_hat as written, and its split (Fz, kz) kept across launches
  // LL-line region of the persistent kernel (B == 1 only; zeroed by cerot_init; offsets depend on B, m and
  // the SM count only, so cerot_init finds it without n, R or the dtype)
  void* ll_base;
  size_t ll_bytes;
  unsigned long long* lepoch;   // [1]
  uint4* zlines;                // [m]
  uint4* rlines;                // [2][lcap]
  uint4* plines;                // [2][lcap][m]
  int lcap;                     // = SM count
  // K-ITER-RES (k_iter_res.cu): integer column sums [3][m] and arrival counters [8] + reduction epoch (u64);
  // inside the LL region, so cerot_init zeroes them too
  unsigned long long* rsum;
  unsigned* rcnt;
};
// Lays the workspace out from `base` (may be NULL to only size it). Returns the byte count. R = rows held
// per problem (m unless row-sharded).
size_t carve_workspace(void* base, int64_t B, int64_t n, int64_t m, int64_t R, int dtype, int sm_count,
                       Workspace* ws);

int device_sm_count();
void set_error(const std::string& msg);

// ------------------------------------------------------------------------------- launchers
// R = rows held per block (-1: m, unsharded)
cudaError_t launch_aggregate(const void* C, int64_t B, int64_t n, int64_t m, int dtype, void* G, int32_t* A,
                             int32_t* nonfinite, cudaStream_t s, int64_t R = -1);
cudaError_t launch_precompute(const void* C, const void* G, int64_t B, int64_t n, int64_t m, int dtype,
                              const double* eps, void* S, cudaStream_t s);
int expand_path(int64_t n, int64_t m, int dtype);
cudaError_t launch_expand(const void* S, const int32_t* A, int64_t B, int64_t n, int64_t m, int dtype, void* out,
                          cudaStream_t s, int64_t R = -1);

struct IterArgs {
  const double* alpha;
  const double* beta;
  const void* C;
  const void* G;
  const double* eps;
  double* w_hat;
  double* z_hat;
  int64_t B, n, m;
  int64_t R;          // rows of each problem held by this call (== m unless row-sharded)
  int64_t row_begin;  // global index of the first held row
  int dtype;
  double tol;
  int64_t check_every;
  uint32_t flags;
};
cudaError_t launch_init(const double* alpha, const double* beta, int64_t B, int64_t m, uint32_t flags, double* z_hat,
                        const Workspace& ws, cudaStream_t s);
// Row pass (p-update + column partials) of one iteration into ws.partials[parity].
cudaError_t launch_rows(const IterArgs& a, const Workspace& ws, const UnitPlan& up, int parity, cudaStream_t s);
// Column pass (deterministic reduction + q-update + monitor) reading ws.partials[parity].
cudaError_t launch_cols(const IterArgs& a, const Workspace& ws, const UnitPlan& up, int parity, cudaStream_t s);
// Up to max_iter iterations of the generic row/column kernels as ONE CUDA graph with a device-side while loop
// (conditional node): the loop ends when every problem is frozen by the freeze rule or after max_iter
// iterations; no host synchronisation in between.
cudaError_t launch_ldg_loop(const IterArgs& a, const Workspace& ws, const UnitPlan& up, int64_t max_iter,
                            cudaStream_t s);
bool tma_eligible(const IterArgs& a, int sms = 0);   // sms: SMs the launch may use (0: all)
// Cluster-resident small problems (fp32, m <= 256, m % 4 == 0): `iters` full iterations of every problem.
bool batch_cluster_eligible(const IterArgs& a);
// m <= 128: one CTA of each cluster runs the whole iteration chain, the others stream the Gibbs terms
// (k_batch_chain.cu); launch_batch_cluster dispatches to it when eligible.
bool batch_chain_eligible(const IterArgs& a);
cudaError_t launch_batch_chain(const IterArgs& a, const Workspace& ws, int iters, cudaStream_t s);
cudaError_t launch_batch_cluster(const IterArgs& a, const Workspace& ws, int iters, cudaStream_t s);
// Persistent TMA kernel: `iters` full iterations (cooperative launch), or the row pass of one iteration
// into ws.partials[parity] when rows_only.
cudaError_t launch_iter_tma(const IterArgs& a, const Workspace& ws, int iters, bool rows_only, int parity,
                            cudaStream_t s);
// Fused multi-GPU row sharding: the persistent kernel of one rank (or, emulated, of all ranks in one
// cooperative grid on one GPU) with the column-sum exchange done in-kernel through peer-mapped LL lines.
struct FusedRank {
  IterArgs a;                          // this rank's shard (row_begin, R)
  Workspace ws;
  uint4* xpeer[kMaxRanks];             // every rank's line array, as addressed by this rank
  unsigned long long* xepoch;          // this rank's epoch counter
  int rank;
  unsigned char* xres[kMaxRanks];      // every rank's K-ITER-RES exchange region, as addressed by this rank
};
// K-ITER-RES (k_iter_res.cu): the iteration of a problem or row shard whose cost fits on chip (TMEM + shared
// memory of one CTA per SM): C3 and the C4 shards of 4- and 8-GPU partitions.
struct ResCfg {
  int h, W, ncl, MR, nq_max, tq, nsq;
  size_t smem;
};
bool res_config(int64_t n, int64_t m, int64_t R, int64_t Rlo, int sms, int nranks_emulated, ResCfg* out);
bool res_eligible(const IterArgs& a, int sms = 0);
cudaError_t launch_iter_res(const IterArgs& a, const Workspace& ws, int iters, cudaStream_t s);
bool res_fused_config(const FusedRank& r, int nranks, bool emulate, ResCfg* c);
cudaError_t launch_iter_res_fused(const FusedRank* r, int nv, int nranks, bool emulate, int iters, cudaStream_t s);
int res_path_h(int64_t n, int64_t m, int64_t R);
int fused_column_slices(int64_t m, int nranks, int sms);
cudaError_t launch_iter_tma_fused(const FusedRank* r, int nv, int nranks, bool emulate, int iters, cudaStream_t s);
// Plan pass over the held rows: T blocks (optional) + unit partials in the workspace (no finalisation).
cudaError_t launch_plan(const IterArgs& a, const Workspace& ws, const UnitPlan& up, void* T_blocks, cudaStream_t s);
// NEXT-3 C-SROT (squared regulariser): one alternating-maximisation sweep (w-step, z-step + monitor), plan.
cudaError_t launch_srot_sweep(const IterArgs& a, const double* gam, const Workspace& ws, cudaStream_t s);
cudaError_t launch_srot_plan(const IterArgs& a, const double* gam, const Workspace& ws, void* T_blocks,
                             double* report, cudaStream_t s);
cudaError_t launch_colsum(const Workspace& ws, const UnitPlan& up, int64_t B, int64_t m, int parity, double* c,
                          cudaStream_t s);
cudaError_t launch_zupdate(const double* c, const double* beta, int64_t B, int64_t m, int64_t n, double tol,
                           int64_t check_every, double* z_hat, const Workspace& ws, cudaStream_t s);
cudaError_t launch_plan_reduce_local(const IterArgs& a, const Workspace& ws, const UnitPlan& up, double* buf,
                                     cudaStream_t s);
cudaError_t launch_plan_finalize_buf(const IterArgs& a, const Workspace& ws, const double* buf, double* report,
                                     cudaStream_t s);

// NEXT-2 (k_full.cu): fold averages, tiling, transposed blocks, stage-2 half-iterations and report
cudaError_t launch_fold(const double* a, const double* b, int64_t n, int64_t m, double* alpha, double* beta,
                        cudaStream_t s);
cudaError_t launch_tile(const double* z, int64_t n, int64_t m, double* g, cudaStream_t s);
cudaError_t launch_transpose_blocks(const void* C, int64_t n, int64_t m, int dtype, void* Bt, cudaStream_t s);
cudaError_t launch_full_pass(const void* X, int64_t n, int64_t m, int dtype, const double* eps, const double* mu,
                             const double* in, double* out, double* dev, double* rep, int mode, cudaStream_t s);
cudaError_t launch_full_monitor(const double* dev, int64_t d, double* out, cudaStream_t s);
cudaError_t launch_full_finalize(const double* rep_rows, const double* rep_cols, const double* a, const double* b,
                                 const double* f, const double* g, int64_t d, const double* eps, double residual,
                                 double* report, cudaStream_t s);

}  // namespace cot
