/*
 * cyclicot.h — C ABI of the B200-native (sm_100a) hot path of
 *   "Optimal Transport with Cyclic Symmetry" (arXiv 2311.13147; /root/reference/PAPER.md = P).
 *
 * Problem (Assumption 1): d = n*m; the marginals are n stacked copies of alpha, beta in
 * R^m_{>0}; the d x d cost is block-circulant, block (r, s) = C_{(s - r) mod n}
 * (P:161-168). Everything here works on the REDUCED data: the n cost blocks C_0..C_{n-1}.
 *
 * Conventions shared by every entry point
 *   - Pointers are caller-owned DEVICE memory unless a comment says HOST. Arrays are dense, row-major,
 *     contiguous; the library never allocates persistent device memory and never frees caller memory.
 *     Scratch lives in a caller-provided workspace of cot_workspace_bytes(...) bytes.
 *   - Layouts (B = number of independent problems in the batch, B >= 1):
 *       C       [B][n][m][m]  cost blocks, block k row-major (C[b][k][i][j] = C_ijk of problem b)
 *       G       [B][m][m]     aggregated cost (same dtype as C);  argmin [B][m][m] int32
 *       alpha   [B][m], beta [B][m]   float64, every entry > 0, sum(alpha_b) == sum(beta_b)
 *                                      (the library checks this to 1e-6 relative; convention 1/n)
 *       eps     [B]           float64 > 0 (the paper's lambda)
 *       w_hat, z_hat [B][m]   float64 SCALED dual potentials w/eps, z/eps
 *       T_full  [B][d][d]     dense plan, same dtype as C
 *   - dtype: COT_F32 (float) or COT_F64 (double) for C, G, S, T.
 *   - stream: a cudaStream_t passed as void*. All work is enqueued on it; calls are asynchronous
 *     unless the comment says "synchronises".
 *   - Every function returns a cot_status. Negative = error (nothing useful was written; the
 *     message is in cot_last_error(), which is thread-local). COT_NOT_CONVERGED (> 0) is a warning:
 *     outputs are valid.
 *   - Reported objective values are FULL-problem scale (x n).
 *   - No CPU fallback: every compute step runs in the sm_100a kernels of this library.
 */
#ifndef CYCLICOT_H
#define CYCLICOT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define COT_ABI_VERSION 1

typedef enum { COT_F32 = 0, COT_F64 = 1 } cot_dtype;

typedef enum {
  COT_OK = 0,
  COT_NOT_CONVERGED = 1,   /* warning: max_iter reached before tol; outputs valid                     */
  COT_E_ARG = -1,          /* n < 1, m < 1, B < 1, NULL required pointer, bad dtype, eps <= 0, ...     */
  COT_E_NONFINITE = -2,    /* a cost entry is NaN or +-Inf                                 */
  COT_E_MARGINAL = -3,     /* alpha_i <= 0, beta_j <= 0, or |sum alpha - sum beta| > 1e-6 relative    */
  COT_E_CUDA = -4,         /* a CUDA runtime error (message in cot_last_error)                         */
  COT_E_NCCL = -5,         /* an NCCL error in the sharded path                                        */
  COT_E_WORKSPACE = -6,    /* ws_bytes < cot_workspace_bytes(...) or misaligned workspace              */
  COT_E_UNDERFLOW = -7,    /* a column sum fell below 1e-28 in the fp32 path (eps too small)*/
  COT_E_PEER = -8          /* fused multi-GPU path: a peer rank's exchange line did not arrive in 20 s */
} cot_status;

/* Flags for cerot_* */
#define COT_COLD_START 0x1u   /* start from q = 1_m, i.e. z_hat = 0 (Alg. 2 line 2); otherwise
                                 z_hat is a warm start                                                  */
#define COT_FORCE_LDG  0x2u   /* use the generic LDG row kernels even where the TMA (large problems)  */
                              /* or cluster-resident (small problems) kernels apply                    */
#define COT_FORCE_TMA  0x8u   /* B == 1 fp32 problems that would run cluster-resident use the persistent  */
                              /* TMA-streaming kernel instead (tests of that kernel on small shapes)     */
#define COT_PRECOMPUTED 0x4u  /* NEXT-1: `C` is S from cerot_precompute ([B][1][m][m], pass n = 1); the   */
                              /* row pass uses s_ij = S_ij instead of re-streaming the n blocks          */
#define COT_DETERMINISTIC 0x10u  /* persistent / fused path (B == 1, fp32): column sums accumulated exactly in    */
                                 /* 128-bit fixed point (2^-120) and row sums in a fixed warp order, so every   */
                                 /* iterate is bitwise identical for any row partition (SM count, 1-8 ranks).   */
                                 /* Needs <= 8 rows per CTA (COT_E_CUDA otherwise) and sum(alpha) < 2^7 (the    */
                                 /* fixed point has 8 integer bits; cerot_state returns COT_E_ARG otherwise).   */
                                 /* Rejected (COT_E_ARG) by the split / NCCL entry points (cerot_rows,          */
                                 /* cerot_rows_shard, cerot_iter_sharded, cerot_solve_sharded).                 */
/* Diagnostic flags (results are NOT valid with them; used by scripts/ubench_iter.py only):          */
#define COT_DIAG_NO_COMPUTE 0x100u  /* TMA kernel: consumers only acknowledge slots (pure HBM stream)    */
#define COT_DIAG_NO_SYNC    0x200u  /* TMA kernel: skip the column pass and device-wide barriers        */
#define COT_DIAG_NO_STREAM  0x400u  /* TMA kernel: stream C in the first iteration only (later k-sums    */
                                    /* read stale slots: wrong results; isolates the sync chain)         */

/* Layout of one problem's report (HOST struct; the device report is the same 8 doubles + 2 ints). */
typedef struct {
  double objective;   /* transport cost n * sum_k <C_k, T_k>       (Table 1 'Obj. value')      */
  double reg_primal;  /* objective + n*eps*sum T (log T - 1)       (eq. problem_CROT)      */
  double dual;        /* n * (<w,alpha> + <z,beta> - eps sum T)    (eq. dual_problem_cyclic_ROT)      */
  double row_l1;      /* || T 1_d - a ||_1 of the full plan                                            */
  double col_l1;      /* || T^T 1_d - b ||_1                                                           */
  double col_l2;      /* || T^T 1_d - b ||_2   (the marginal error of Sec. 6.1)                */
  double mass;        /* sum of the full plan                                                          */
  double residual;    /* last convergence monitor n*sum_j|c_j - beta_j| after a p-update */
  int64_t iters;      /* iterations performed                                                          */
  int32_t converged;  /* 1 if the monitor reached tol                                                  */
  int32_t status;     /* per-problem cot_status                                                        */
} cot_report;

int cot_abi_version(void);
const char* cot_last_error(void);
/* Select the CUDA device every later call of this thread runs on (cudaSetDevice in the library's own, statically
 * linked runtime). Optional: by default the library uses the device whose context is current on the thread
 * (e.g. the one torch.cuda.set_device selected). Returns COT_E_CUDA for an invalid ordinal. */
int cot_set_device(int device);

/* Bytes of scratch needed by cerot_* for this shape on the current device (includes G and argmin for
 * cerot_solve, the fp64 column partials, the per-problem solver state and the plan reductions). */
size_t cot_workspace_bytes(int64_t B, int64_t n, int64_t m, int dtype);

/* ---------------------------------------------------------------------------------------------- */
/* A2  C-LOT aggregation (Alg. 1 line 1).                                                   */
/*   G[b][i][j] = min_k C[b][k][i][j]            (eq. definition_G)                       */
/*   argmin[b][i][j] = the SMALLEST k attaining it (tie remark P:291); G is the value stored   */
/*   at that k, so the sign of zero is deterministic. Comparisons only: bit-exact.                    */
/*   d_nonfinite (DEVICE int32, may be NULL): receives the number of NaN/Inf entries of C (it is     */
/*   overwritten, not accumulated). Asynchronous; use cot_check_nonfinite to turn it into a status.   */
int clot_aggregate(const void* C, int64_t B, int64_t n, int64_t m, int dtype,
                   void* G, int32_t* argmin, int32_t* d_nonfinite, void* stream);

/* NEXT-1 (Alg. 2 line 1 as written): S[b][i][j] = sum_k exp((G_ij - C_ijk)/eps_b) in [1, n]       */
/* (the cyclic Gibbs kernel K_ij = S_ij exp(-G_ij/eps), eq. def_Kij, kept G-shifted). Then       */
/* cerot_iter(C = S, n = 1, flags | COT_PRECOMPUTED) runs O(m^2) iterations. Asynchronous.         */
int cerot_precompute(const void* C, const void* G, int64_t B, int64_t n, int64_t m, int dtype, const double* eps,
                     void* S, void* stream);

/* Synchronises `stream`, reads *d_nonfinite and returns COT_E_NONFINITE if it is > 0, else COT_OK. */
int cot_check_nonfinite(const int32_t* d_nonfinite, void* stream);

/* A6  Dense d x d block-circulant expansion (Lemma 1, eq. blkstr_optimal_solution).      */
/*   argmin != NULL  (C-LOT, Alg. 1 lines 3-6): S is [B][m][m];                           */
/*       T_full[b][r*m+i][s*m+j] = S[b][i][j] if argmin[b][i][j] == (s - r) mod n, else 0            */
/*       (the lift of eq. optimal_solution_problem_CLOT, placed by Lemma 1).               */
/*   argmin == NULL  (C-EROT blocks, Alg. 2 line 10): S is T_blocks [B][n][m][m];              */
/*       T_full[b][r*m+i][s*m+j] = T_blocks[b][(s - r) mod n][i][j].                                   */
/*   Pure placement: bit-exact copies. T_full must hold B*d*d elements.                               */
int clot_expand(const void* S, const int32_t* argmin, int64_t B, int64_t n, int64_t m, int dtype,
                void* T_full, void* stream);
/* Which expansion kernel clot_expand / clot_expand_shard select for (n, m, dtype) (introspection for tests   */
/* and profiling; no device work): 2 = whole dense rows assembled in shared memory (small n*m), 1 = one       */
/* m-segment per unit written by n TMA bulk stores (m*esize % 16 == 0, m*esize <= 32 KiB), 0 = vector stores  */
/* (ragged m). -1 on bad arguments.                                                                           */
int cot_expand_path(int64_t n, int64_t m, int dtype);

/* ---------------------------------------------------------------------------------------------- */
/* A3+A4  Cyclic Sinkhorn iterations (Alg. 2 lines 3-6) in the log domain of             */
/* eq. optimal_f_sinkhorn_logdomain. One iteration = p-update then q-update:            */
/*   for each row i:  s_ij = sum_k exp((G_ij - C_ijk)/eps)            (streamed, never cached)      */
/*                    x_ij = z_hat_j - G_ij/eps,  M_i = max_j x_ij                                  */
/*                    r_i = sum_j s_ij exp(x_ij - M_i)                                              */
/*                    w_hat_i = log alpha_i - M_i - log r_i                                         */
/*   for each column: c_j = sum_i (alpha_i/r_i) s_ij exp(x_ij - M_i)   (plan column sum after p)    */
/*                    z_hat_j += log beta_j - log c_j                  (q-update)            */
/*                    monitor  n * sum_j |c_j - beta_j|                   */
/* G must be clot_aggregate's output for the same C (it is the exact per-(i,j) maximum of -C/eps).  */
/* cerot_init: resets the solver state in `workspace` (iteration counters, convergence flags) and,  */
/*   with COT_COLD_START, sets z_hat = 0 (q = 1_m). It validates alpha, beta on the device;   */
/*   a violation is reported by cerot_state / cerot_solve as COT_E_MARGINAL.                          */
/* cerot_iter: enqueues exactly `iters` iterations (asynchronous). With tol > 0, a problem whose      */
/*   monitor is <= tol at an iteration t with t % check_every == 0 is frozen after that iteration's  */
/*   q-update (its potentials stop changing), exactly as the oracle's stopping rule.                 */
int cerot_init(const double* alpha, const double* beta, int64_t B, int64_t m, uint32_t flags,
               double* z_hat, void* workspace, size_t ws_bytes, void* stream);
int cerot_iter(const double* alpha, const double* beta, const void* C, const void* G,
               int64_t B, int64_t n, int64_t m, int dtype, const double* eps,
               int64_t iters, double tol, int64_t check_every, uint32_t flags,
               double* w_hat, double* z_hat, void* workspace, size_t ws_bytes, void* stream);
/* Which kernel cerot_iter / cerot_solve run for this shape (no device work): 0 = generic row/column      */
/* kernels (k_rows_ldg + k_cols, one launch pair per iteration), 1 = the persistent TMA-streaming kernel  */
/* (k_iter_tma: B == 1, fp32, m % 4 == 0, m <= 1024; HBM-bound), 2 = the cluster-resident kernel          */
/* (k_batch_cluster: fp32, m % 4 == 0, 8 <= m <= 256; whole problem on chip, SFU-bound), 3 = the          */
/* cluster-resident chain kernel (k_batch_chain: fp32, m % 4 == 0, m <= 128; one CTA per cluster runs the  */
/* iteration chain, the others stream the Gibbs terms; COT_BATCH_CHAIN=0 in the environment disables it);  */
/* 4 = the on-chip-resident kernel (k_iter_res: B == 1, fp32, m % 128 == 0, m <= 1024, the n*m^2 costs fit */
/* in the TMEM + shared memory of one CTA per SM, e.g. C3; SFU-bound; COT_RES=0 in the environment        */
/* disables it; not with COT_DETERMINISTIC, COT_PRECOMPUTED, COT_FORCE_TMA or COT_FORCE_LDG);              */
/* -1: bad shape.                                                                                          */
int cot_iter_path(int64_t B, int64_t n, int64_t m, int dtype, uint32_t flags);
/* The kernel cerot_iter_fused runs for a rank holding R rows of an nranks-way balanced row partition of a */
/* fp32 problem: 4 = k_iter_res (the rank's shard fits on chip: the C4 shards of 8-GPU    */
/* partitions), 1 = k_iter_tma (the streaming persistent kernel); emulated = 1 asks for the one-GPU       */
/* emulation (cerot_iter_fused_emulated: each virtual rank on 1/nranks of the SMs). -1: bad arguments.     */
int cot_fused_path(int64_t n, int64_t m, int64_t R, int nranks, int emulated, uint32_t flags);
/* The two halves of one cerot_iter iteration, for callers that interleave work between them (the
 * row-sharded multi-GPU path reduces the column sums across ranks in between; bench.py times the row
 * pass alone). `parity` (0/1) selects the column-partial buffer; use the iteration index & 1.
 *   cerot_rows: the p-update of every held row + fp64 column partials (the streamed n*m^2 pass).
 *   cerot_cols: deterministic column reduction, q-update, monitor and freeze rule.                    */
int cerot_rows(const double* alpha, const void* C, const void* G, int64_t B, int64_t n, int64_t m, int dtype,
               const double* eps, uint32_t flags, const double* z_hat, double* w_hat,
               void* workspace, size_t ws_bytes, int parity, void* stream);
int cerot_cols(const double* beta, int64_t B, int64_t n, int64_t m, int dtype, double tol, int64_t check_every,
               double* z_hat, void* workspace, size_t ws_bytes, int parity, void* stream);

/* Synchronises `stream` and copies the per-problem state to HOST arrays (any may be NULL):         */
/*   iters_done[B] (int64), converged[B] (int32), residual[B] (double). Returns COT_E_MARGINAL,     */
/*   COT_E_UNDERFLOW if the device flagged one, else COT_OK.                                          */
int cerot_state(const void* workspace, int64_t B, int64_t m, int64_t n, int dtype,
                int64_t* iters_done, int32_t* converged, double* residual, void* stream);

/* A5  Plan reconstruction (Alg. 2 lines 7-9; eq. optimality_condition):     */
/*   T[b][k][i][j] = exp(w_hat_i + z_hat_j - C_ijk/eps)  written if T_blocks != NULL, and the       */
/*   fp64 reductions of cot_report (objective, reg_primal, dual, row/col residuals, mass) written    */
/*   to d_report (DEVICE, [B][8] doubles in cot_report field order; may be NULL). Asynchronous.       */
int cerot_plan(const double* alpha, const double* beta, const void* C, const void* G,
               int64_t B, int64_t n, int64_t m, int dtype, const double* eps,
               const double* w_hat, const double* z_hat, void* T_blocks, double* d_report,
               void* workspace, size_t ws_bytes, void* stream);

/* Whole C-EROT solve (A2..A5): clot_aggregate into the workspace, cerot_init, then up to max_iter   */
/* iterations with the freeze rule applied ON THE DEVICE every check_every iterations ("until        */
/* convergence"): one persistent launch (cluster-resident / TMA kernels), or one CUDA graph    */
/* with a device-side while loop (generic kernels) -- no host round trip per check -- then cerot_plan.*/
/* Synchronises once, for the report.                                                                */
/* report: HOST array of B cot_report. T_blocks may be NULL. Returns COT_OK, COT_NOT_CONVERGED if    */
/* some problem did not reach tol (tol > 0), or an error.                                             */
int cerot_solve(const double* alpha, const double* beta, const void* C,
                int64_t B, int64_t n, int64_t m, int dtype, const double* eps,
                double tol, int64_t max_iter, int64_t check_every, uint32_t flags,
                double* w_hat, double* z_hat, void* T_blocks,
                void* workspace, size_t ws_bytes, cot_report* report, void* stream);

/* ---------------------------------------------------------------------------------------------- */
/* Row sharding across GPUs (B == 1). GPU g holds rows [row_begin, row_begin + R) of every */
/* block: C_local [n][R][m], G_local [R][m] (clot_aggregate of C_local with m columns and R rows, i.e.    */
/* call it with the shard viewed as [n][R][m] -- see paper_2311_13147_b200.dist), while alpha, beta,     */
/* w_hat, z_hat stay full length [m] (w_hat is written only on the held rows; z_hat is replicated).       */
/* The p-update of the held rows is local; the plan column sums are summed across GPUs with ONE           */
/* m-length fp64 ncclAllReduce per iteration; every GPU then applies the identical q-update. NCCL is     */
/* loaded at run time (libnccl.so.2, the copy torch uses); `comm` == NULL means a single GPU.            */
size_t cot_workspace_bytes_sharded(int64_t n, int64_t m, int64_t R, int dtype);
/* G, argmin of the held rows: C_local [n][R][m] -> G_local, argmin_local [R][m] (as clot_aggregate). */
int clot_aggregate_shard(const void* C_local, int64_t n, int64_t R, int64_t m, int dtype, void* G_local,
                         int32_t* argmin_local, int32_t* d_nonfinite, void* stream);
/* The held rows of the dense d x d plan: T_rows [n][R][d], row (r, i) = full-plan row r*m + row_begin + i  */
/* (as clot_expand; S_local = argmin_local ? S [R][m] : T_local [n][R][m]).                              */
int clot_expand_shard(const void* S_local, const int32_t* argmin_local, int64_t n, int64_t R, int64_t m, int dtype,
                      void* T_rows, void* stream);
/* Writes a new 128-byte ncclUniqueId to id128 (HOST memory; broadcast it to every rank). */
int cot_nccl_unique_id(void* id128);
/* Creates the communicator of `rank` among `nranks` (ncclCommInitRank; current CUDA device). Owned by    */
/* the caller; release with cot_comm_destroy.                                                            */
int cot_comm_init(const void* id128, int nranks, int rank, void** comm);
int cot_comm_destroy(void* comm);
/* Row pass of one iteration on the held rows + their column sums c_local[m] (DEVICE, fp64; not yet      */
/* reduced across GPUs).                                                                                  */
int cerot_rows_shard(const double* alpha, const void* C_local, const void* G_local, int64_t n, int64_t m,
                     int64_t row_begin, int64_t R, int dtype, const double* eps, uint32_t flags,
                     const double* z_hat, double* w_hat, double* c_local, void* workspace, size_t ws_bytes,
                     void* stream);
/* q-update from the fully reduced column sums c[m] (DEVICE): z_hat_j += log beta_j - log c_j, monitor,    */
/* iteration count and freeze rule in the workspace state.                                               */
int cerot_zupdate(const double* beta, const double* c, int64_t n, int64_t m, double tol, int64_t check_every,
                  double* z_hat, void* workspace, size_t ws_bytes, void* stream);
/* `iters` iterations: cerot_rows_shard -> ncclAllReduce(c) (if comm) -> cerot_zupdate, all on `stream`.  */
/* Groups of 8 iterations are captured once as a CUDA graph (on a private stream) and replayed on      */
/* `stream`; bitwise the same as per-iteration launches (COT_SHARDED_NO_GRAPH=1 forces those). The       */
/* caller's comm must not be used by another thread while this call enqueues.                           */
int cerot_iter_sharded(const double* alpha, const double* beta, const void* C_local, const void* G_local,
                       int64_t n, int64_t m, int64_t row_begin, int64_t R, int dtype, const double* eps,
                       int64_t iters, double tol, int64_t check_every, uint32_t flags, double* w_hat,
                       double* z_hat, void* workspace, size_t ws_bytes, void* comm, void* stream);
/* Plan of the held rows (T_local [n][R][m] if non-NULL) + report reduced across GPUs (identical on every */
/* GPU; d_report DEVICE [8] doubles, cot_report field order).                                            */
int cerot_plan_sharded(const double* alpha, const double* beta, const void* C_local, const void* G_local,
                       int64_t n, int64_t m, int64_t row_begin, int64_t R, int dtype, const double* eps,
                       const double* w_hat, const double* z_hat, void* T_local, double* d_report,
                       void* workspace, size_t ws_bytes, void* comm, void* stream);

/* The whole solve of this rank: clot_aggregate of the held rows (into the workspace), cold  */
/* start, cerot_iter_sharded in chunks of check_every with the freeze rule when tol > 0, then the   */
/* plan of the held rows (T_local [n][R][m] if non-NULL) and the report reduced across ranks (HOST,       */
/* identical on every rank). Synchronises. COT_NOT_CONVERGED if tol > 0 was not reached.                 */
int cerot_solve_sharded(const double* alpha, const double* beta, const void* C_local, int64_t n, int64_t m,
                        int64_t row_begin, int64_t R, int dtype, const double* eps, double tol, int64_t max_iter,
                        int64_t check_every, uint32_t flags, double* w_hat, double* z_hat, void* T_local,
                        void* workspace, size_t ws_bytes, void* comm, cot_report* report, void* stream);

/* ---------------------------------------------------------------------------------------------- */
/* Fused row sharding: the same partition and arithmetic as cerot_iter_sharded, but the    */
/* exchange step runs INSIDE the persistent iteration kernel (one cooperative launch per rank for all     */
/* `iters` iterations): after the local row pass of iteration t (Alg. 2 line 4), CTA b of every    */
/* rank writes its rank's column sums of column slice b straight into every rank's exchange buffer over  */
/* NVLink (peer-mapped CUDA IPC memory; 16-byte LL lines carrying the iteration's generation, no fence), */
/* then reads all ranks' lines of slice b from its own buffer and sums them in rank order, so c_j and the */
/* q-update (Alg. 2 line 5) are bitwise identical on every rank. No NCCL call and no host          */
/* round trip per iteration. Requirements: fp32 C, m % 4 == 0, m <= 1024, nranks <= COT_MAX_RANKS, a     */
/* balanced contiguous row partition (R = floor or ceil of m / nranks; any R when nranks == 1, which runs */
/* one shard alone with the exchange to itself), every rank launching the same                          */
/* `iters` (a peer that never arrives makes the call's state report COT_E_PEER after 20 s).              */
#define COT_MAX_RANKS 8
/* Bytes of one rank's exchange buffer: a 256-byte header (the iteration epoch) + [2][nranks][m] lines.  */
size_t cot_xchg_bytes(int64_t m, int nranks);
/* Allocates and zeroes this rank's exchange buffer (cudaMalloc on the current device; the library owns  */
/* it until cot_xchg_free) and, if ipc_handle != NULL, writes its 64-byte cudaIpcMemHandle (HOST) for the */
/* other ranks.                                                                                           */
int cot_xchg_alloc(int64_t m, int nranks, void** xbuf, void* ipc_handle);
/* Maps another rank's exchange buffer (64-byte handle from its cot_xchg_alloc) into this process with    */
/* peer access; release with cot_xchg_close. Never call it on this rank's own handle.                     */
int cot_xchg_open(const void* ipc_handle, void** peer_xbuf);
int cot_xchg_close(void* peer_xbuf);
int cot_xchg_free(void* xbuf);
/* The same exchange buffers as NCCL symmetric memory (NCCL >= 2.27 device API; for processes where CUDA   */
/* IPC handles cannot be shared): COLLECTIVE over `comm` (cot_comm_init) -- every rank allocates its       */
/* cot_xchg_bytes(m, nranks) buffer with ncclMemAlloc (zeroed) and registers it with                       */
/* ncclCommWindowRegister(NCCL_WIN_COLL_SYMMETRIC); *xbuf = this rank's buffer (DEVICE), *win = the window. */
/* cot_xchg_nccl_peers writes (HOST array [nranks]) the device address of every rank's copy as mapped into */
/* this process (the window's load/store-accessible peer pointers: ncclGetPeerPointer), i.e. the xbufs of  */
/* cerot_iter_fused. cot_xchg_nccl_free deregisters (collective) and frees. COT_E_NCCL if the loaded NCCL  */
/* has no symmetric-memory API or the registration fails.                                                  */
int cot_xchg_nccl_alloc(void* comm, int64_t m, int nranks, void** xbuf, void** win);
int cot_xchg_nccl_peers(void* win, int nranks, void** peers);
int cot_xchg_nccl_free(void* comm, void* xbuf, void* win);
/* `iters` fused iterations of this rank. xbufs: HOST array [nranks] of DEVICE pointers, rank q's         */
/* exchange buffer as addressed by this process (xbufs[rank] = own buffer). Other arguments and the       */
/* state / potentials as cerot_iter_sharded; cerot_init first (per rank). Asynchronous.                  */
int cerot_iter_fused(const double* alpha, const double* beta, const void* C_local, const void* G_local,
                     int64_t n, int64_t m, int64_t row_begin, int64_t R, int dtype, const double* eps,
                     int64_t iters, double tol, int64_t check_every, uint32_t flags, double* w_hat,
                     double* z_hat, void* workspace, size_t ws_bytes, int nranks, int rank, void* const* xbufs,
                     void* stream);
/* Emulation on ONE GPU (the recipe for testing a multi-rank protocol without the GPUs): all `nranks`    */
/* ranks' fused iterations in ONE cooperative launch, each virtual rank on 1/nranks of the SMs with its   */
/* own shard, workspace, potentials and exchange buffer (all on this device). Every per-rank argument is  */
/* a HOST array [nranks]; alpha, beta, eps are shared.                                                   */
int cerot_iter_fused_emulated(int nranks, const double* alpha, const double* beta, const void* const* C_local,
                              const void* const* G_local, int64_t n, int64_t m, const int64_t* row_begin,
                              const int64_t* R, int dtype, const double* eps, int64_t iters, double tol,
                              int64_t check_every, uint32_t flags, double* const* w_hat, double* const* z_hat,
                              void* const* workspace, const size_t* ws_bytes, void* const* xbufs, void* stream);

/* ---------------------------------------------------------------------------------------------- */
/* NEXT-2: the two-stage Sinkhorn algorithm for C-EROT with APPROXIMATE cyclic symmetry (Algorithm 3,    */
/* P:457-484). a, b: DEVICE [d] fp64 (d = n*m; in the simplex, only approximately n-periodic); C: DEVICE  */
/* [n][m][m] the blocks of the strictly block-circulant cost; eps DEVICE [1].                    */
/*   stage 1 (lines 2-10): alpha, beta = fold averages of a, b, cyclic Sinkhorn of the hot   */
/*     path from q^ = 1 for iters1 iterations or until its monitor (n*sum|c - beta|) <= tol1;  */
/*     w_hat, z_hat DEVICE [m] receive its eps-scaled potentials;                                         */
/*   stage 2 (lines 11-16): the original Sinkhorn on the explicit d x d problem from g = concatenated     */
/*     z_hat, without materialising the d x d cost (each CTA stages the n block rows C_k[i][:] once and   */
/*     serves the n rows r*m + i); iters2 iterations or until sum_J |T^T 1 - b|_J of the row-exact plan   */
/*     <= tol2 (checked every check_every); f_hat, g_hat DEVICE [d] eps-scaled potentials (out).         */
/*   report (HOST, FULL-problem values, no factor n): transport cost, regularised primal, dual, marginal  */
/*     residuals and mass of T = diag(p) K diag(q) (line 17); iters_done HOST [2] = stage-1, stage-2      */
/*     iterations. Synchronises. Returns COT_NOT_CONVERGED if tol2 > 0 was not reached.                   */
size_t cot_two_stage_workspace_bytes(int64_t n, int64_t m, int dtype);
int cerot_two_stage(const double* a, const double* b, const void* C, int64_t n, int64_t m, int dtype,
                    const double* eps, int64_t iters1, double tol1, int64_t iters2, double tol2,
                    int64_t check_every, double* f_hat, double* g_hat, double* w_hat, double* z_hat,
                    void* workspace, size_t ws_bytes, cot_report* report, int64_t* iters_done, void* stream);
/* The same algorithm with App. F's stage-2 stopping rule: stage 2 runs until the difference     */
/* between its objective function value and `obj_ref` -- the value obtained by directly solving the       */
/* problem with the original Sinkhorn algorithm, supplied by the caller (HOST double) -- is below         */
/* `tol_obj` (> 0; the paper uses 1e-4), checked every check_every iterations on the plan                 */
/* T = diag(p) K diag(q) after the iteration's q-update, or for iters2 iterations. The objective is the   */
/* regularised primal <C,T> + eps sum T (log T - 1) (report->reg_primal, FULL-problem value; DESIGN       */
/* reading Q19). Each check costs the two report passes of one extra iteration and one host sync.         */
/* report->residual receives the last measured |objective - obj_ref| (0 if never checked). Returns        */
/* COT_NOT_CONVERGED if the gap was not reached, COT_E_ARG if tol_obj <= 0 or obj_ref is not finite.      */
/* Other arguments, workspace and outputs as cerot_two_stage.                                             */
int cerot_two_stage_gap(const double* a, const double* b, const void* C, int64_t n, int64_t m, int dtype,
                        const double* eps, int64_t iters1, double tol1, int64_t iters2, double obj_ref,
                        double tol_obj, int64_t check_every, double* f_hat, double* g_hat, double* w_hat,
                        double* z_hat, void* workspace, size_t ws_bytes, cot_report* report, int64_t* iters_done,
                        void* stream);

/* ---------------------------------------------------------------------------------------------- */
/* NEXT-4: the small LOT of Theorem 1 (eq. small_problem_CLOT; Alg. 1 line 2), the paper's     */
/* serial step, on the HOST: min <G, S> s.t. S 1 = alpha, S^T 1 = beta, S >= 0 by the primal network     */
/* simplex method with exact integer flows (masses scaled to 2^50) and the       */
/* strongly feasible pivot rule. All pointers HOST, row-major fp64: alpha, beta [m] (> 0, equal sums to  */
/* 1e-6 relative), G [m][m] finite; outputs S [m][m] (a vertex: <= 2m-1 non-zeros), *value = <G, S>, and  */
/* (optional, may be NULL) dual potentials u, v [m] with u_i + v_j <= G_ij, equality where S_ij > 0, and  */
/* the pivot count. Synchronous, single-threaded, no device work; thread-safe on distinct buffers.        */
int clot_small_lot(const double* alpha, const double* beta, const double* G, int64_t m, double* S,
                   double* value, double* u, double* v, int64_t* pivots);
/* The C-LOT value of the explicit d x d problem (Theorem 1, at full scale): value_full = n * <G, S*> */
/* with S* from clot_small_lot (written to S, HOST [m][m]); value_small = <G, S*> (may be NULL). HOST, synchronous. */
int clot_lot_value(const double* alpha, const double* beta, const double* G, int64_t m, int64_t n, double* S,
                   double* value_full, double* value_small);

/* ---------------------------------------------------------------------------------------------- */
/* NEXT-3: C-SROT, strongly convex regularised OT through the 2m-variable Fenchel dual        */
/* (Theorem 2) by alternating maximisation: each sweep solves every w_i with z fixed, then     */
/* every z_j with w fixed, by safeguarded Newton on the monotone derivative; the plan is      */
/* T_ijk = (phi*)'(w_i + z_j - C_ijk). Regulariser COT_REG_SQUARED: phi(x) = x^2/(2 gamma)    */
/* for x >= 0, (phi*)'(y) = gamma max(y, 0) (sparse plans). reg_param: DEVICE [B] gamma. w, z: DEVICE      */
/* [B][m] fp64 in cost units (not eps-scaled); cold start z = 0 with COT_COLD_START. Stops when the       */
/* monitor n*sum_j|c_j - beta_j| (plan after the w-step) <= tol, checked every check_every sweeps, or    */
/* after max_sweeps. report: HOST [B]. Synchronises.                                                      */
typedef enum { COT_REG_ENTROPIC = 0, COT_REG_SQUARED = 1 } cot_reg;
int csrot_solve(const double* alpha, const double* beta, const void* C, int64_t B, int64_t n, int64_t m, int dtype,
                int reg, const double* reg_param, double tol, int64_t max_sweeps, int64_t check_every,
                uint32_t flags, double* w, double* z, void* T_blocks, void* workspace, size_t ws_bytes,
                cot_report* report, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CYCLICOT_H */
