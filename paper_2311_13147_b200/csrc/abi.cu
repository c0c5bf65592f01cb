// C ABI of libcyclicot (include/cyclicot.h): argument validation, workspace carving, launch sequencing and
// the NCCL communicator of the row-sharded path. No compute happens here: every step of the path is one of
// the kernels in k_*.cu (or an NCCL collective between them).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nccl_device.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

namespace cot {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

int device_sm_count() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) return 148;
  return sms;
}

UnitPlan unit_plan(int64_t B, int64_t R, int sm_count) {
  UnitPlan up;
  const int64_t rows = B * R;
  int64_t rpu = (rows + sm_count - 1) / sm_count;   // ~ one unit per SM
  if (rpu < 1) rpu = 1;
  if (rpu > R) rpu = R;
  up.rpu = rpu;
  up.upp = (R + rpu - 1) / rpu;
  up.U = B * up.upp;
  const int64_t cap = (int64_t)sm_count * 4;
  up.grid = (int)std::min<int64_t>(up.U, cap);
  return up;
}

static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

size_t carve_workspace(void* base, int64_t B, int64_t n, int64_t m, int64_t R, int dtype, int sm_count,
                       Workspace* ws) {
  (void)n;
  const UnitPlan up = unit_plan(B, R, sm_count);
  const size_t esz = dtype == COT_F32 ? 4 : 8;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 256);
    return base ? static_cast<char*>(base) + o : nullptr;
  };
  // Order matters: the per-problem state comes first so its offset depends on B only (cerot_init and
  // cerot_state find it without knowing n, R or the dtype); the dtype-sized G comes last.
  Workspace w{};
  w.state = reinterpret_cast<SolverState*>(take((size_t)B * sizeof(SolverState)));
  w.counters = reinterpret_cast<unsigned*>(take((size_t)B * 4));
  w.grid_bar = reinterpret_cast<unsigned*>(take(16));
  w.loopctl = reinterpret_cast<unsigned*>(take(16));
  w.nonfinite = reinterpret_cast<int32_t*>(take(4));
  w.report = reinterpret_cast<double*>(take((size_t)B * kReportDoubles * 8));
  // monitor partials: per 32-column tile (k_cols, k_zupdate) or per 4-column tile (C-SROT z-step)
  w.resid_part = reinterpret_cast<double*>(take((size_t)std::max<int64_t>(B * ((m + 3) / 4), sm_count) * 8));
  if (B == 1) {   // LL lines of the persistent kernel
    const size_t o0 = off;
    w.lepoch = reinterpret_cast<unsigned long long*>(take(256));
    w.zlines = reinterpret_cast<uint4*>(take((size_t)m * 16));
    w.rlines = reinterpret_cast<uint4*>(take((size_t)2 * sm_count * 16));
    w.plines = reinterpret_cast<uint4*>(take((size_t)2 * sm_count * (2 * m) * 16));   // 2 lines / value (deterministic)
    w.lcap = sm_count;
    w.rcnt = reinterpret_cast<unsigned*>(take(64));
    w.rsum = reinterpret_cast<unsigned long long*>(take((size_t)3 * m * 8));
    w.ll_base = base ? static_cast<char*>(base) + o0 : nullptr;
    w.ll_bytes = off - o0;
  }
  w.plan_scal = reinterpret_cast<double*>(take((size_t)up.U * kPlanScalars * 8));
  w.partials[0] = reinterpret_cast<double*>(take((size_t)(up.U * m) * 8));
  w.partials[1] = reinterpret_cast<double*>(take((size_t)(up.U * m) * 8));
  w.c_local = reinterpret_cast<double*>(take((size_t)(B * m) * 8));
  w.c_global = reinterpret_cast<double*>(take((size_t)(B * m) * 8));
  w.plan_buf = reinterpret_cast<double*>(take((size_t)(B * (kPlanBufHead + m)) * 8));
  w.rowscal = reinterpret_cast<double*>(take((size_t)(B * m * 4) * 8));
  w.zcache = reinterpret_cast<double*>(take((size_t)(B * m * 3) * 8));
  w.A = reinterpret_cast<int32_t*>(take((size_t)(B * R * m) * 4));
  w.G = take((size_t)(B * R * m) * esz);
  if (ws) *ws = w;
  return off;
}

// ------------------------------------------------------------------------------------------- NCCL
// NCCL is loaded at run time (the copy torch already loaded when present): the library itself loads and
// runs on one GPU without it; only the communicator functions need it.
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  // NCCL >= 2.27 symmetric memory (optional): the fused exchange over NCCL-registered windows
  ncclResult_t (*MemAlloc)(void**, size_t) = nullptr;
  ncclResult_t (*MemFree)(void*) = nullptr;
  ncclResult_t (*CommWindowRegister)(ncclComm_t, void*, size_t, ncclWindow_t*, int) = nullptr;
  ncclResult_t (*CommWindowDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
};
static NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.err = std::string("cannot load libnccl.so.2: ") + (e ? e : "unknown error");
      return;
    }
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    api.MemAlloc = (decltype(api.MemAlloc))dlsym(h, "ncclMemAlloc");
    api.MemFree = (decltype(api.MemFree))dlsym(h, "ncclMemFree");
    api.CommWindowRegister = (decltype(api.CommWindowRegister))dlsym(h, "ncclCommWindowRegister");
    api.CommWindowDeregister = (decltype(api.CommWindowDeregister))dlsym(h, "ncclCommWindowDeregister");
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.GetErrorString;
    if (!api.ok) api.err = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

// Device addresses of every rank's copy of an NCCL symmetric window (header-only device API: the window's LSA
// flat base + rank stride), written to out[0 .. nranks)
__global__ void k_window_peers(ncclWindow_t w, int nranks, void** out) {
  if (threadIdx.x == 0 && blockIdx.x == 0)
    for (int r = 0; r < nranks; ++r) out[r] = ncclGetPeerPointer(w, 0, r);
}

size_t xchg_res_offset(int64_t m, int nranks) {
  return kXchgHeader + (size_t)2 * nranks * (2 * m) * sizeof(uint4);   // 2 lines per value in the deterministic mode
}
}  // namespace cot

using namespace cot;

#define COT_CHECK_CUDA(expr)                                                      \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) {                                                      \
      set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));              \
      return COT_E_CUDA;                                                          \
    }                                                                             \
  } while (0)

#define COT_CHECK_NCCL(expr)                                                      \
  do {                                                                            \
    ncclResult_t _r = (expr);                                                     \
    if (_r != ncclSuccess) {                                                      \
      set_error(std::string(#expr) + ": " + nccl_api().GetErrorString(_r));          \
      return COT_E_NCCL;                                                          \
    }                                                                             \
  } while (0)

static int arg_error(const std::string& m) {
  set_error(m);
  return COT_E_ARG;
}

static int check_shape(int64_t B, int64_t n, int64_t m, int dtype) {
  if (B < 1 || n < 1 || m < 1) return arg_error("B, n, m must be >= 1");
  if (dtype != COT_F32 && dtype != COT_F64) return arg_error("dtype must be COT_F32 or COT_F64");
  if (m > 8192) return arg_error("m > 8192 is not supported by the row kernels");
  if (n > (1 << 24)) return arg_error("n too large");
  return COT_OK;
}

static int check_ws(void* workspace, size_t ws_bytes, int64_t B, int64_t n, int64_t m, int64_t R, int dtype,
                    Workspace* ws) {
  const size_t need = carve_workspace(nullptr, B, n, m, R, dtype, device_sm_count(), nullptr);
  if (!workspace || ws_bytes < need) {
    set_error("workspace too small: need " + std::to_string(need) + " bytes, got " + std::to_string(ws_bytes));
    return COT_E_WORKSPACE;
  }
  if (reinterpret_cast<uintptr_t>(workspace) % 256 != 0) {
    set_error("workspace must be 256-byte aligned");
    return COT_E_WORKSPACE;
  }
  carve_workspace(workspace, B, n, m, R, dtype, device_sm_count(), ws);
  return COT_OK;
}

static IterArgs make_args(const double* alpha, const double* beta, const void* C, const void* G, int64_t B, int64_t n,
                          int64_t m, int dtype, const double* eps, double tol, int64_t check_every, uint32_t flags,
                          double* w_hat, double* z_hat, int64_t row_begin = 0, int64_t R = -1) {
  IterArgs a;
  a.alpha = alpha;
  a.beta = beta;
  a.C = C;
  a.G = G;
  a.eps = eps;
  a.w_hat = w_hat;
  a.z_hat = z_hat;
  a.B = B;
  a.n = n;
  a.m = m;
  a.R = R < 0 ? m : R;
  a.row_begin = row_begin;
  a.dtype = dtype;
  a.tol = tol;
  a.check_every = check_every > 0 ? check_every : 1;
  a.flags = flags;
  return a;
}

// One iteration of the row pass into ws.partials[parity] on the held rows (TMA rows-only or LDG).
static cudaError_t rows_pass(const IterArgs& a, const Workspace& ws, int parity, cudaStream_t s) {
  if (tma_eligible(a)) return launch_iter_tma(a, ws, 1, true, parity & 1, s);
  return launch_rows(a, ws, unit_plan(a.B, a.R, device_sm_count()), parity & 1, s);
}

// Plan pass + local reductions (+ allreduce over comm when given) + report.
static int plan_and_report(const IterArgs& a, const Workspace& ws, void* T_blocks, double* d_report, void* comm,
                           cudaStream_t s) {
  const UnitPlan up = unit_plan(a.B, a.R, device_sm_count());
  COT_CHECK_CUDA(launch_plan(a, ws, up, T_blocks, s));
  COT_CHECK_CUDA(launch_plan_reduce_local(a, ws, up, ws.plan_buf, s));
  if (comm) {
    COT_CHECK_NCCL(nccl_api().AllReduce(ws.plan_buf, ws.plan_buf, (size_t)(a.B * (kPlanBufHead + a.m)), ncclFloat64,
                                    ncclSum, (ncclComm_t)comm, s));
  }
  COT_CHECK_CUDA(launch_plan_finalize_buf(a, ws, ws.plan_buf, d_report ? d_report : ws.report, s));
  return COT_OK;
}

extern "C" {

int cot_abi_version(void) { return COT_ABI_VERSION; }

const char* cot_last_error(void) { return g_last_error.c_str(); }

int cot_set_device(int device) {
  COT_CHECK_CUDA(cudaSetDevice(device));
  return COT_OK;
}

size_t cot_workspace_bytes(int64_t B, int64_t n, int64_t m, int dtype) {
  if (B < 1 || n < 1 || m < 1) return 0;
  return carve_workspace(nullptr, B, n, m, m, dtype, device_sm_count(), nullptr);
}

size_t cot_workspace_bytes_sharded(int64_t n, int64_t m, int64_t R, int dtype) {
  if (n < 1 || m < 1 || R < 1 || R > m) return 0;
  return carve_workspace(nullptr, 1, n, m, R, dtype, device_sm_count(), nullptr);
}

int clot_aggregate(const void* C, int64_t B, int64_t n, int64_t m, int dtype, void* G, int32_t* argmin,
                   int32_t* d_nonfinite, void* stream) {
  int st = check_shape(B, n, m, dtype);
  if (st) return st;
  if (!C || !G || !argmin) return arg_error("clot_aggregate: C, G and argmin must be non-NULL");
  COT_CHECK_CUDA(launch_aggregate(C, B, n, m, dtype, G, argmin, d_nonfinite, (cudaStream_t)stream));
  return COT_OK;
}

int cerot_precompute(const void* C, const void* G, int64_t B, int64_t n, int64_t m, int dtype, const double* eps,
                     void* S, void* stream) {
  int st = check_shape(B, n, m, dtype);
  if (st) return st;
  if (!C || !G || !eps || !S) return arg_error("cerot_precompute: NULL argument");
  COT_CHECK_CUDA(launch_precompute(C, G, B, n, m, dtype, eps, S, (cudaStream_t)stream));
  return COT_OK;
}

int cot_check_nonfinite(const int32_t* d_nonfinite, void* stream) {
  if (!d_nonfinite) return arg_error("cot_check_nonfinite: NULL flag");
  int32_t h = 0;
  COT_CHECK_CUDA(cudaMemcpyAsync(&h, d_nonfinite, sizeof(h), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  COT_CHECK_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  if (h > 0) {
    set_error(std::to_string(h) + " non-finite cost entries");
    return COT_E_NONFINITE;
  }
  return COT_OK;
}

int clot_expand(const void* S, const int32_t* argmin, int64_t B, int64_t n, int64_t m, int dtype, void* T_full,
                void* stream) {
  int st = check_shape(B, n, m, dtype);
  if (st) return st;
  if (!S || !T_full) return arg_error("clot_expand: S and T_full must be non-NULL");
  COT_CHECK_CUDA(launch_expand(S, argmin, B, n, m, dtype, T_full, (cudaStream_t)stream));
  return COT_OK;
}

int cerot_init(const double* alpha, const double* beta, int64_t B, int64_t m, uint32_t flags, double* z_hat,
               void* workspace, size_t ws_bytes, void* stream) {
  if (B < 1 || m < 1) return arg_error("B, m must be >= 1");
  if (!alpha || !beta || !z_hat) return arg_error("cerot_init: alpha, beta, z_hat must be non-NULL");
  // the state block is at the start of the workspace for every (n, R, dtype) (see carve_workspace)
  Workspace ws;
  const size_t need = (size_t)B * (sizeof(SolverState) + 4) + 2048;
  if (!workspace || ws_bytes < need) {
    set_error("workspace too small");
    return COT_E_WORKSPACE;
  }
  carve_workspace(workspace, B, 1, m, m, COT_F32, device_sm_count(), &ws);
  if (ws.ll_base && static_cast<char*>(ws.ll_base) + ws.ll_bytes > static_cast<char*>(workspace) + ws_bytes) {
    set_error("workspace too small");
    return COT_E_WORKSPACE;
  }
  if (ws.ll_base) COT_CHECK_CUDA(cudaMemsetAsync(ws.ll_base, 0, ws.ll_bytes, (cudaStream_t)stream));
  COT_CHECK_CUDA(launch_init(alpha, beta, B, m, flags, z_hat, ws, (cudaStream_t)stream));
  return COT_OK;
}

int cerot_iter(const double* alpha, const double* beta, const void* C, const void* G, int64_t B, int64_t n, int64_t m,
               int dtype, const double* eps, int64_t iters, double tol, int64_t check_every, uint32_t flags,
               double* w_hat, double* z_hat, void* workspace, size_t ws_bytes, void* stream) {
  int st = check_shape(B, n, m, dtype);
  if (st) return st;
  if (!alpha || !beta || !C || !G || !eps || !w_hat || !z_hat) return arg_error("cerot_iter: NULL argument");
  if (iters < 0 || tol < 0 || !(tol == tol)) return arg_error("cerot_iter: iters >= 0 and tol >= 0 required");
  Workspace ws;
  st = check_ws(workspace, ws_bytes, B, n, m, m, dtype, &ws);
  if (st) return st;
  const IterArgs a = make_args(alpha, beta, C, G, B, n, m, dtype, eps, tol, check_every, flags, w_hat, z_hat);
  const UnitPlan up = unit_plan(B, m, device_sm_count());
  cudaStream_t s = (cudaStream_t)stream;
  if (iters > 0 && batch_cluster_eligible(a)) {   // small problems: whole problem on chip (C5, C2)
    COT_CHECK_CUDA(launch_batch_cluster(a, ws, (int)iters, s));
    return COT_OK;
  }
  if (iters > 0 && res_eligible(a)) {              // cost fits on chip (C3): TMEM + shared-memory resident
    COT_CHECK_CUDA(launch_iter_res(a, ws, (int)iters, s));
    return COT_OK;
  }
  if (iters > 0 && tma_eligible(a)) {              // large problem: persistent TMA stream (C4)
    COT_CHECK_CUDA(launch_iter_tma(a, ws, (int)iters, false, 0, s));
    return COT_OK;
  }
  for (int64_t t = 0; t < iters; ++t) {
    COT_CHECK_CUDA(launch_rows(a, ws, up, (int)(t & 1), s));
    COT_CHECK_CUDA(launch_cols(a, ws, up, (int)(t & 1), s));
  }
  return COT_OK;
}

int cot_expand_path(int64_t n, int64_t m, int dtype) {
  if (n < 1 || m < 1 || (dtype != COT_F32 && dtype != COT_F64)) return -1;
  return expand_path(n, m, dtype);
}

int cot_iter_path(int64_t B, int64_t n, int64_t m, int dtype, uint32_t flags) {
  if (B < 1 || n < 1 || m < 1) return -1;
  const IterArgs a = make_args(nullptr, nullptr, nullptr, nullptr, B, n, m, dtype, nullptr, 0.0, 1, flags, nullptr,
                               nullptr);
  if (batch_chain_eligible(a)) return 3;
  if (batch_cluster_eligible(a)) return 2;
  if (res_eligible(a)) return 4;
  if (tma_eligible(a)) return 1;
  return 0;
}

int cot_fused_path(int64_t n, int64_t m, int64_t R, int nranks, int emulated, uint32_t flags) {
  if (n < 1 || m < 1 || R < 1 || R > m || nranks < 1 || nranks > kMaxRanks) return -1;
  FusedRank fr{};
  fr.a = make_args(nullptr, nullptr, nullptr, nullptr, 1, n, m, COT_F32, nullptr, 0.0, 1, flags, nullptr, nullptr, 0,
                   R);
  for (int q = 0; q < nranks; ++q) fr.xres[q] = reinterpret_cast<unsigned char*>(1);   // shape query only
  return res_fused_config(fr, nranks, emulated != 0, nullptr) ? 4 : 1;
}

int cerot_rows(const double* alpha, const void* C, const void* G, int64_t B, int64_t n, int64_t m, int dtype,
               const double* eps, uint32_t flags, const double* z_hat, double* w_hat, void* workspace,
               size_t ws_bytes, int parity, void* stream) {
  int st = check_shape(B, n, m, dtype);
  if (st) return st;
  if (flags & COT_DETERMINISTIC)
    return arg_error("cerot_rows: COT_DETERMINISTIC is implemented by the persistent kernel only (cerot_iter, "
                     "cerot_iter_fused); the split row pass has no fixed-point partials");
  if (!alpha || !C || !G || !eps || !w_hat || !z_hat) return arg_error("cerot_rows: NULL argument");
  Workspace ws;
  st = check_ws(workspace, ws_bytes, B, n, m, m, dtype, &ws);
  if (st) return st;
  const IterArgs a = make_args(alpha, nullptr, C, G, B, n, m, dtype, eps, 0.0, 1, flags, w_hat,
                               const_cast<double*>(z_hat));
  COT_CHECK_CUDA(rows_pass(a, ws, parity, (cudaStream_t)stream));
  return COT_OK;
}

int cerot_cols(const double* beta, int64_t B, int64_t n, int64_t m, int dtype, double tol, int64_t check_every,
               double* z_hat, void* workspace, size_t ws_bytes, int parity, void* stream) {
  int st = check_shape(B, n, m, dtype);
  if (st) return st;
  if (!beta || !z_hat) return arg_error("cerot_cols: NULL argument");
  if (tol < 0) return arg_error("cerot_cols: tol >= 0 required");
  Workspace ws;
  st = check_ws(workspace, ws_bytes, B, n, m, m, dtype, &ws);
  if (st) return st;
  const IterArgs a = make_args(nullptr, beta, nullptr, nullptr, B, n, m, dtype, nullptr, tol, check_every, 0, nullptr,
                               z_hat);
  COT_CHECK_CUDA(launch_cols(a, ws, unit_plan(B, m, device_sm_count()), parity & 1, (cudaStream_t)stream));
  return COT_OK;
}

int cerot_state(const void* workspace, int64_t B, int64_t m, int64_t n, int dtype, int64_t* iters_done,
                int32_t* converged, double* residual, void* stream) {
  if (B < 1 || m < 1 || !workspace) return arg_error("cerot_state: bad arguments");
  Workspace ws;
  carve_workspace(const_cast<void*>(workspace), B, n, m, m, dtype, device_sm_count(), &ws);
  std::vector<SolverState> h((size_t)B);
  COT_CHECK_CUDA(cudaMemcpyAsync(h.data(), ws.state, (size_t)B * sizeof(SolverState), cudaMemcpyDeviceToHost,
                                 (cudaStream_t)stream));
  COT_CHECK_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  int flags = 0;
  for (int64_t b = 0; b < B; ++b) {
    if (iters_done) iters_done[b] = h[b].iters;
    if (converged) converged[b] = h[b].converged;
    if (residual) residual[b] = h[b].residual;
    flags |= h[b].flags;
  }
  if (flags & STATE_BAD_MARGINAL) {
    set_error("alpha/beta must be > 0 with equal sums (1e-6 relative)");
    return COT_E_MARGINAL;
  }
  if (flags & STATE_UNDERFLOW) {
    set_error("a column sum fell below 1e-28 (fp32 underflow; eps too small for this cost scale)");
    return COT_E_UNDERFLOW;
  }
  if (flags & STATE_DET_REFUSED) {
    set_error("COT_DETERMINISTIC needs sum(alpha) < 2^7 (128-bit fixed point with 120 fraction bits); "
              "rescale alpha and beta");
    return COT_E_ARG;
  }
  if (flags & STATE_PEER_TIMEOUT) {
    set_error("fused multi-GPU path: a peer rank's exchange line did not arrive within 20 s");
    return COT_E_PEER;
  }
  return COT_OK;
}

int cerot_plan(const double* alpha, const double* beta, const void* C, const void* G, int64_t B, int64_t n, int64_t m,
               int dtype, const double* eps, const double* w_hat, const double* z_hat, void* T_blocks,
               double* d_report, void* workspace, size_t ws_bytes, void* stream) {
  int st = check_shape(B, n, m, dtype);
  if (st) return st;
  if (!alpha || !beta || !C || !G || !eps || !w_hat || !z_hat) return arg_error("cerot_plan: NULL argument");
  Workspace ws;
  st = check_ws(workspace, ws_bytes, B, n, m, m, dtype, &ws);
  if (st) return st;
  IterArgs a = make_args(alpha, beta, C, G, B, n, m, dtype, eps, 0.0, 1, 0, const_cast<double*>(w_hat),
                         const_cast<double*>(z_hat));
  return plan_and_report(a, ws, T_blocks, d_report, nullptr, (cudaStream_t)stream);
}

int cerot_solve(const double* alpha, const double* beta, const void* C, int64_t B, int64_t n, int64_t m, int dtype,
                const double* eps, double tol, int64_t max_iter, int64_t check_every, uint32_t flags, double* w_hat,
                double* z_hat, void* T_blocks, void* workspace, size_t ws_bytes, cot_report* report, void* stream) {
  int st = check_shape(B, n, m, dtype);
  if (st) return st;
  if (!alpha || !beta || !C || !eps || !w_hat || !z_hat || !report) return arg_error("cerot_solve: NULL argument");
  if (max_iter < 0 || tol < 0) return arg_error("cerot_solve: max_iter >= 0 and tol >= 0 required");
  Workspace ws;
  st = check_ws(workspace, ws_bytes, B, n, m, m, dtype, &ws);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (check_every < 1) check_every = 1;
  // A2: G and argmin (G is the exact per-(i,j) max of -C/eps used by the row kernel)
  COT_CHECK_CUDA(launch_aggregate(C, B, n, m, dtype, ws.G, ws.A, ws.nonfinite, s));
  st = cot_check_nonfinite(ws.nonfinite, stream);
  if (st) return st;
  COT_CHECK_CUDA(launch_init(alpha, beta, B, m, flags, z_hat, ws, s));
  const IterArgs a = make_args(alpha, beta, C, ws.G, B, n, m, dtype, eps, tol, check_every, flags, w_hat, z_hat);
  const UnitPlan up = unit_plan(B, m, device_sm_count());
  std::vector<int64_t> it((size_t)B);
  std::vector<int32_t> conv((size_t)B);
  std::vector<double> res((size_t)B);
  // "Until convergence" (Alg. 2 line 6) on the device: the persistent kernels run up to max_iter iterations
  // in one launch and apply the freeze rule themselves; the generic kernels run as one CUDA graph
  // with a device-side while loop. No host round trip until the report.
  if (max_iter > 0) {
    if (batch_cluster_eligible(a) || res_eligible(a) || tma_eligible(a)) {
      for (int64_t done = 0; done < max_iter;) {   // int-sized launches (one launch unless max_iter >= 2^31)
        const int chunk = (int)std::min<int64_t>(max_iter - done, 0x7fffffff);
        if (batch_cluster_eligible(a))
          COT_CHECK_CUDA(launch_batch_cluster(a, ws, chunk, s));
        else if (res_eligible(a))
          COT_CHECK_CUDA(launch_iter_res(a, ws, chunk, s));
        else
          COT_CHECK_CUDA(launch_iter_tma(a, ws, chunk, false, 0, s));
        done += chunk;
      }
    } else {
      COT_CHECK_CUDA(launch_ldg_loop(a, ws, up, max_iter, s));
    }
  }
  st = plan_and_report(a, ws, T_blocks, ws.report, nullptr, s);
  if (st) return st;
  std::vector<double> rep((size_t)B * kReportDoubles);
  COT_CHECK_CUDA(cudaMemcpyAsync(rep.data(), ws.report, rep.size() * 8, cudaMemcpyDeviceToHost, s));
  st = cerot_state(workspace, B, m, n, dtype, it.data(), conv.data(), res.data(), stream);
  if (st) return st;
  bool all_conv = true;
  for (int64_t b = 0; b < B; ++b) {
    cot_report& r = report[b];
    const double* d = rep.data() + b * kReportDoubles;
    r.objective = d[0];
    r.reg_primal = d[1];
    r.dual = d[2];
    r.row_l1 = d[3];
    r.col_l1 = d[4];
    r.col_l2 = d[5];
    r.mass = d[6];
    r.residual = d[7];
    r.iters = it[(size_t)b];
    r.converged = conv[(size_t)b];
    r.status = (tol > 0.0 && !conv[(size_t)b]) ? COT_NOT_CONVERGED : COT_OK;
    all_conv = all_conv && (r.status == COT_OK);
  }
  return all_conv ? COT_OK : COT_NOT_CONVERGED;
}

// ------------------------------------------------------------------------------------- NEXT-2: two-stage
static size_t two_stage_layout(int64_t n, int64_t m, int dtype, char* base, size_t* off_red, double** alpha,
                               double** beta, void** Bt, double** dev, double** mon, double** rep_rows,
                               double** rep_cols, double** report) {
  const size_t esz = dtype == COT_F32 ? 4 : 8;
  const int64_t d = n * m;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = (off + bytes + 255) / 256 * 256;
    return base ? base + o : nullptr;
  };
  *off_red = off;
  take(carve_workspace(nullptr, 1, n, m, m, dtype, device_sm_count(), nullptr));
  *alpha = reinterpret_cast<double*>(take((size_t)m * 8));
  *beta = reinterpret_cast<double*>(take((size_t)m * 8));
  *Bt = take((size_t)n * m * m * esz);
  *dev = reinterpret_cast<double*>(take((size_t)d * 8));
  *mon = reinterpret_cast<double*>(take(8));
  *rep_rows = reinterpret_cast<double*>(take((size_t)3 * d * 8));
  *rep_cols = reinterpret_cast<double*>(take((size_t)3 * d * 8));
  *report = reinterpret_cast<double*>(take(kReportDoubles * 8));
  return off;
}

// Reduced C-EROT iterations on one problem with the state checks of cerot_solve; returns COT_* status.
static int iterate_reduced(const IterArgs& a, const Workspace& ws, void* workspace, int64_t n, int64_t m, int dtype,
                           int64_t max_iter, double tol, int64_t check_every, cudaStream_t s) {
  const UnitPlan up = unit_plan(1, m, device_sm_count());
  int64_t done = 0;
  int64_t it = 0;
  int32_t conv = 0;
  double res = 0.0;
  while (done < max_iter) {
    const int64_t chunk = std::min<int64_t>(check_every, max_iter - done);
    if (batch_cluster_eligible(a)) {
      COT_CHECK_CUDA(launch_batch_cluster(a, ws, (int)chunk, s));
    } else if (res_eligible(a)) {
      COT_CHECK_CUDA(launch_iter_res(a, ws, (int)chunk, s));
    } else if (tma_eligible(a)) {
      COT_CHECK_CUDA(launch_iter_tma(a, ws, (int)chunk, false, 0, s));
    } else {
      for (int64_t t = 0; t < chunk; ++t) {
        COT_CHECK_CUDA(launch_rows(a, ws, up, (int)((done + t) & 1), s));
        COT_CHECK_CUDA(launch_cols(a, ws, up, (int)((done + t) & 1), s));
      }
    }
    done += chunk;
    if (tol > 0.0) {
      const int st = cerot_state(workspace, 1, m, n, dtype, &it, &conv, &res, s);
      if (st) return st;
      if (conv) break;
    }
  }
  return COT_OK;
}

size_t cot_two_stage_workspace_bytes(int64_t n, int64_t m, int dtype) {
  if (n < 1 || m < 1 || (dtype != COT_F32 && dtype != COT_F64)) return 0;
  size_t o;
  double *al, *be, *dv, *mo, *rr, *rc, *rp;
  void* bt;
  return two_stage_layout(n, m, dtype, nullptr, &o, &al, &be, &bt, &dv, &mo, &rr, &rc, &rp);
}

// Both stage-2 stopping rules: the marginal monitor (tol2) and App. F's objective gap (tol_obj > 0: |regularised
// primal of the current plan - obj_ref| < tol_obj), each checked every check_every iterations.
static int two_stage_impl(const double* a, const double* b, const void* C, int64_t n, int64_t m, int dtype,
                          const double* eps, int64_t iters1, double tol1, int64_t iters2, double tol2, double obj_ref,
                          double tol_obj, int64_t check_every, double* f_hat, double* g_hat, double* w_hat,
                          double* z_hat, void* workspace, size_t ws_bytes, cot_report* report, int64_t* iters_done,
                          void* stream) {
  int st = check_shape(1, n, m, dtype);
  if (st) return st;
  if (!a || !b || !C || !eps || !f_hat || !g_hat || !w_hat || !z_hat)
    return arg_error("cerot_two_stage: NULL argument");
  if (iters1 < 0 || iters2 < 0 || tol1 < 0 || tol2 < 0) return arg_error("cerot_two_stage: negative count or tol");
  if (check_every < 1) check_every = 1;
  const size_t need = cot_two_stage_workspace_bytes(n, m, dtype);
  if (!workspace || ws_bytes < need || reinterpret_cast<uintptr_t>(workspace) % 256) {
    set_error("cerot_two_stage: workspace too small or misaligned: need " + std::to_string(need));
    return COT_E_WORKSPACE;
  }
  cudaStream_t s = (cudaStream_t)stream;
  char* base = static_cast<char*>(workspace);
  size_t off_red;
  double *alpha, *beta, *dev, *mon, *rep_rows, *rep_cols, *rep;
  void* Bt;
  two_stage_layout(n, m, dtype, base, &off_red, &alpha, &beta, &Bt, &dev, &mon, &rep_rows, &rep_cols, &rep);
  void* red = base + off_red;
  const size_t red_bytes = carve_workspace(nullptr, 1, n, m, m, dtype, device_sm_count(), nullptr);
  Workspace ws;
  carve_workspace(red, 1, n, m, m, dtype, device_sm_count(), &ws);
  const int64_t d = n * m;
  // ---- stage 1 (Alg. 3 lines 2-10): fold averages, then the cyclic Sinkhorn of the hot path
  COT_CHECK_CUDA(launch_fold(a, b, n, m, alpha, beta, s));
  COT_CHECK_CUDA(launch_aggregate(C, 1, n, m, dtype, ws.G, ws.A, ws.nonfinite, s));
  st = cot_check_nonfinite(ws.nonfinite, stream);
  if (st) return st;
  st = cerot_init(alpha, beta, 1, m, COT_COLD_START, z_hat, red, red_bytes, stream);
  if (st) return st;
  const IterArgs ia = make_args(alpha, beta, C, ws.G, 1, n, m, dtype, eps, tol1, check_every, 0, w_hat, z_hat);
  st = iterate_reduced(ia, ws, red, n, m, dtype, iters1, tol1, check_every, s);
  if (st) return st;
  int64_t it1 = 0;
  int32_t conv1 = 0;
  double res1 = 0.0;
  st = cerot_state(red, 1, m, n, dtype, &it1, &conv1, &res1, stream);
  if (st) return st;
  // ---- stage 2 (lines 11-16): g = concatenated z_hat, then the original Sinkhorn on the explicit problem
  COT_CHECK_CUDA(launch_tile(z_hat, n, m, g_hat, s));
  COT_CHECK_CUDA(launch_transpose_blocks(C, n, m, dtype, Bt, s));
  int64_t it2 = 0;
  double residual = 0.0;
  bool have_res = false, gap_ok = false;
  double gap = 0.0;
  for (int64_t t = 0; t < iters2; ++t) {
    COT_CHECK_CUDA(launch_full_pass(C, n, m, dtype, eps, a, g_hat, f_hat, nullptr, nullptr, 0, s));   // p-update
    COT_CHECK_CUDA(launch_full_pass(Bt, n, m, dtype, eps, b, f_hat, g_hat, dev, nullptr, 1, s));     // q-update
    ++it2;
    const bool check = (tol2 > 0.0 && it2 % check_every == 0) || t == iters2 - 1;
    if (check) {
      COT_CHECK_CUDA(launch_full_monitor(dev, d, mon, s));
      COT_CHECK_CUDA(cudaMemcpyAsync(&residual, mon, 8, cudaMemcpyDeviceToHost, s));
      COT_CHECK_CUDA(cudaStreamSynchronize(s));
      have_res = true;
      if (tol2 > 0.0 && it2 % check_every == 0 && residual <= tol2) break;
    }
    if (tol_obj > 0.0 && it2 % check_every == 0) {   // App. F: the objective of the plan after this iteration
      COT_CHECK_CUDA(launch_full_pass(C, n, m, dtype, eps, a, g_hat, f_hat, nullptr, rep_rows, 2, s));
      COT_CHECK_CUDA(launch_full_pass(Bt, n, m, dtype, eps, b, f_hat, g_hat, nullptr, rep_cols, 2, s));
      COT_CHECK_CUDA(launch_full_finalize(rep_rows, rep_cols, a, b, f_hat, g_hat, d, eps, 0.0, rep, s));
      double hv[kReportDoubles];
      COT_CHECK_CUDA(cudaMemcpyAsync(hv, rep, sizeof(hv), cudaMemcpyDeviceToHost, s));
      COT_CHECK_CUDA(cudaStreamSynchronize(s));
      gap = std::fabs(hv[1] - obj_ref);
      if (gap < tol_obj) {
        gap_ok = true;
        break;
      }
    }
  }
  // ---- report of the returned plan T = diag(p) K diag(q) (line 17)
  COT_CHECK_CUDA(launch_full_pass(C, n, m, dtype, eps, a, g_hat, f_hat, nullptr, rep_rows, 2, s));
  COT_CHECK_CUDA(launch_full_pass(Bt, n, m, dtype, eps, b, f_hat, g_hat, nullptr, rep_cols, 2, s));
  COT_CHECK_CUDA(launch_full_finalize(rep_rows, rep_cols, a, b, f_hat, g_hat, d, eps, have_res ? residual : res1,
                                      rep, s));
  double h[kReportDoubles];
  COT_CHECK_CUDA(cudaMemcpyAsync(h, rep, sizeof(h), cudaMemcpyDeviceToHost, s));
  COT_CHECK_CUDA(cudaStreamSynchronize(s));
  const bool wanted = tol2 > 0.0 || tol_obj > 0.0;
  const bool conv = (tol2 > 0.0 && have_res && residual <= tol2) || gap_ok;
  if (report) {
    report->objective = h[0];
    report->reg_primal = h[1];
    report->dual = h[2];
    report->row_l1 = h[3];
    report->col_l1 = h[4];
    report->col_l2 = h[5];
    report->mass = h[6];
    report->residual = tol_obj > 0.0 ? gap : h[7];
    report->iters = it2;
    report->converged = conv;
    report->status = (wanted && !conv) ? COT_NOT_CONVERGED : COT_OK;
  }
  if (iters_done) {
    iters_done[0] = it1;
    iters_done[1] = it2;
  }
  return (wanted && !conv) ? COT_NOT_CONVERGED : COT_OK;
}

int cerot_two_stage(const double* a, const double* b, const void* C, int64_t n, int64_t m, int dtype, const double* eps,
                    int64_t iters1, double tol1, int64_t iters2, double tol2, int64_t check_every, double* f_hat,
                    double* g_hat, double* w_hat, double* z_hat, void* workspace, size_t ws_bytes,
                    cot_report* report, int64_t* iters_done, void* stream) {
  return two_stage_impl(a, b, C, n, m, dtype, eps, iters1, tol1, iters2, tol2, 0.0, 0.0, check_every, f_hat, g_hat,
                        w_hat, z_hat, workspace, ws_bytes, report, iters_done, stream);
}

int cerot_two_stage_gap(const double* a, const double* b, const void* C, int64_t n, int64_t m, int dtype,
                        const double* eps, int64_t iters1, double tol1, int64_t iters2, double obj_ref, double tol_obj,
                        int64_t check_every, double* f_hat, double* g_hat, double* w_hat, double* z_hat,
                        void* workspace, size_t ws_bytes, cot_report* report, int64_t* iters_done, void* stream) {
  if (!(tol_obj > 0.0) || !std::isfinite(obj_ref))
    return arg_error("cerot_two_stage_gap: tol_obj > 0 and a finite obj_ref required");
  return two_stage_impl(a, b, C, n, m, dtype, eps, iters1, tol1, iters2, 0.0, obj_ref, tol_obj, check_every, f_hat,
                        g_hat, w_hat, z_hat, workspace, ws_bytes, report, iters_done, stream);
}

// ------------------------------------------------------------------------------------- NEXT-3: C-SROT
int csrot_solve(const double* alpha, const double* beta, const void* C, int64_t B, int64_t n, int64_t m, int dtype,
                int reg, const double* reg_param, double tol, int64_t max_sweeps, int64_t check_every, uint32_t flags,
                double* w, double* z, void* T_blocks, void* workspace, size_t ws_bytes, cot_report* report,
                void* stream) {
  int st = check_shape(B, n, m, dtype);
  if (st) return st;
  if (reg != COT_REG_SQUARED) return arg_error("csrot_solve: only COT_REG_SQUARED here (entropic: cerot_solve)");
  if (!alpha || !beta || !C || !reg_param || !w || !z || !report) return arg_error("csrot_solve: NULL argument");
  if (max_sweeps < 0 || tol < 0) return arg_error("csrot_solve: max_sweeps >= 0 and tol >= 0 required");
  Workspace ws;
  st = check_ws(workspace, ws_bytes, B, n, m, m, dtype, &ws);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (check_every < 1) check_every = 1;
  COT_CHECK_CUDA(launch_aggregate(C, B, n, m, dtype, ws.G, ws.A, ws.nonfinite, s));   // finiteness check
  st = cot_check_nonfinite(ws.nonfinite, stream);
  if (st) return st;
  COT_CHECK_CUDA(launch_init(alpha, beta, B, m, flags, z, ws, s));
  const IterArgs a = make_args(alpha, beta, C, nullptr, B, n, m, dtype, nullptr, tol, check_every, flags, w, z);
  std::vector<int64_t> it((size_t)B);
  std::vector<int32_t> conv((size_t)B);
  std::vector<double> res((size_t)B);
  int64_t done = 0;
  while (done < max_sweeps) {
    const int64_t chunk = std::min<int64_t>(check_every, max_sweeps - done);
    for (int64_t t = 0; t < chunk; ++t) COT_CHECK_CUDA(launch_srot_sweep(a, reg_param, ws, s));
    done += chunk;
    if (tol > 0.0) {
      st = cerot_state(workspace, B, m, n, dtype, it.data(), conv.data(), res.data(), stream);
      if (st) return st;
      bool all = true;
      for (int64_t b = 0; b < B && all; ++b) all = conv[(size_t)b] != 0;
      if (all) break;
    }
  }
  COT_CHECK_CUDA(launch_srot_plan(a, reg_param, ws, T_blocks, ws.report, s));
  std::vector<double> rep((size_t)B * kReportDoubles);
  COT_CHECK_CUDA(cudaMemcpyAsync(rep.data(), ws.report, rep.size() * 8, cudaMemcpyDeviceToHost, s));
  st = cerot_state(workspace, B, m, n, dtype, it.data(), conv.data(), res.data(), stream);
  if (st) return st;
  bool all_conv = true;
  for (int64_t b = 0; b < B; ++b) {
    cot_report& r = report[b];
    const double* d = rep.data() + b * kReportDoubles;
    r.objective = d[0];
    r.reg_primal = d[1];
    r.dual = d[2];
    r.row_l1 = d[3];
    r.col_l1 = d[4];
    r.col_l2 = d[5];
    r.mass = d[6];
    r.residual = d[7];
    r.iters = it[(size_t)b];
    r.converged = conv[(size_t)b];
    r.status = (tol > 0.0 && !conv[(size_t)b]) ? COT_NOT_CONVERGED : COT_OK;
    all_conv = all_conv && (r.status == COT_OK);
  }
  return all_conv ? COT_OK : COT_NOT_CONVERGED;
}

// ------------------------------------------------------------------------------------- row sharding
int cot_nccl_unique_id(void* id128) {
  if (!id128) return arg_error("cot_nccl_unique_id: NULL output");
  if (!nccl_api().ok) {
    set_error(nccl_api().err);
    return COT_E_NCCL;
  }
  ncclUniqueId id;
  COT_CHECK_NCCL(nccl_api().GetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  memcpy(id128, &id, sizeof(id));
  return COT_OK;
}

int cot_comm_init(const void* id128, int nranks, int rank, void** comm) {
  if (!id128 || !comm || nranks < 1 || rank < 0 || rank >= nranks) return arg_error("cot_comm_init: bad arguments");
  if (!nccl_api().ok) {
    set_error(nccl_api().err);
    return COT_E_NCCL;
  }
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t c = nullptr;
  COT_CHECK_NCCL(nccl_api().CommInitRank(&c, nranks, id, rank));
  *comm = c;
  return COT_OK;
}

int cot_xchg_nccl_alloc(void* comm, int64_t m, int nranks, void** xbuf, void** win) {
  const size_t bytes = cot_xchg_bytes(m, nranks);
  if (!comm || !bytes || !xbuf || !win) return arg_error("cot_xchg_nccl_alloc: need comm, m >= 1, 1 <= nranks <= 8, outputs");
  if (!nccl_api().ok) {
    set_error(nccl_api().err);
    return COT_E_NCCL;
  }
  if (!nccl_api().MemAlloc || !nccl_api().CommWindowRegister) {
    set_error("cot_xchg_nccl_alloc: the loaded NCCL has no symmetric-memory API (ncclMemAlloc / ncclCommWindowRegister)");
    return COT_E_NCCL;
  }
  const size_t padded = (bytes + 4095) / 4096 * 4096;   // NCCL_WIN_REQUIRED_ALIGNMENT
  void* p = nullptr;
  COT_CHECK_NCCL(nccl_api().MemAlloc(&p, padded));
  cudaError_t e = cudaMemset(p, 0, padded);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    nccl_api().MemFree(p);
    set_error(std::string("cot_xchg_nccl_alloc: ") + cudaGetErrorString(e));
    return COT_E_CUDA;
  }
  ncclWindow_t w = nullptr;
  const ncclResult_t r = nccl_api().CommWindowRegister((ncclComm_t)comm, p, padded, &w, NCCL_WIN_COLL_SYMMETRIC);
  if (r != ncclSuccess) {
    nccl_api().MemFree(p);
    set_error(std::string("ncclCommWindowRegister: ") + nccl_api().GetErrorString(r));
    return COT_E_NCCL;
  }
  *xbuf = p;
  *win = (void*)w;
  return COT_OK;
}

int cot_xchg_nccl_peers(void* win, int nranks, void** peers) {
  if (!win || nranks < 1 || nranks > kMaxRanks || !peers) return arg_error("cot_xchg_nccl_peers: bad argument");
  void** d = nullptr;
  COT_CHECK_CUDA(cudaMalloc(&d, sizeof(void*) * kMaxRanks));
  k_window_peers<<<1, 32>>>((ncclWindow_t)win, nranks, d);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(peers, d, sizeof(void*) * nranks, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) {
    set_error(std::string("cot_xchg_nccl_peers: ") + cudaGetErrorString(e));
    return COT_E_CUDA;
  }
  return COT_OK;
}

int cot_xchg_nccl_free(void* comm, void* xbuf, void* win) {
  if (!nccl_api().ok) {
    set_error(nccl_api().err);
    return COT_E_NCCL;
  }
  if (comm && win && nccl_api().CommWindowDeregister)
    COT_CHECK_NCCL(nccl_api().CommWindowDeregister((ncclComm_t)comm, (ncclWindow_t)win));
  if (xbuf && nccl_api().MemFree) COT_CHECK_NCCL(nccl_api().MemFree(xbuf));
  return COT_OK;
}

int cot_comm_destroy(void* comm) {
  if (!comm) return COT_OK;
  if (!nccl_api().ok) {
    set_error(nccl_api().err);
    return COT_E_NCCL;
  }
  COT_CHECK_NCCL(nccl_api().CommDestroy((ncclComm_t)comm));
  return COT_OK;
}

int clot_aggregate_shard(const void* C_local, int64_t n, int64_t R, int64_t m, int dtype, void* G_local,
                         int32_t* argmin_local, int32_t* d_nonfinite, void* stream) {
  int st = check_shape(1, n, m, dtype);
  if (st) return st;
  if (R < 1 || R > m) return arg_error("clot_aggregate_shard: 1 <= R <= m required");
  if (!C_local || !G_local || !argmin_local) return arg_error("clot_aggregate_shard: NULL argument");
  COT_CHECK_CUDA(launch_aggregate(C_local, 1, n, m, dtype, G_local, argmin_local, d_nonfinite, (cudaStream_t)stream, R));
  return COT_OK;
}

int clot_expand_shard(const void* S_local, const int32_t* argmin_local, int64_t n, int64_t R, int64_t m, int dtype,
                      void* T_rows, void* stream) {
  int st = check_shape(1, n, m, dtype);
  if (st) return st;
  if (R < 1 || R > m) return arg_error("clot_expand_shard: 1 <= R <= m required");
  if (!S_local || !T_rows) return arg_error("clot_expand_shard: NULL argument");
  COT_CHECK_CUDA(launch_expand(S_local, argmin_local, 1, n, m, dtype, T_rows, (cudaStream_t)stream, R));
  return COT_OK;
}

int cerot_rows_shard(const double* alpha, const void* C_local, const void* G_local, int64_t n, int64_t m,
                     int64_t row_begin, int64_t R, int dtype, const double* eps, uint32_t flags, const double* z_hat,
                     double* w_hat, double* c_local, void* workspace, size_t ws_bytes, void* stream) {
  int st = check_shape(1, n, m, dtype);
  if (st) return st;
  if (flags & COT_DETERMINISTIC)
    return arg_error("cerot_rows_shard: COT_DETERMINISTIC is implemented by the persistent kernel only (cerot_iter, "
                     "cerot_iter_fused); the split row pass has no fixed-point partials");
  if (R < 1 || row_begin < 0 || row_begin + R > m) return arg_error("cerot_rows_shard: bad row range");
  if (!alpha || !C_local || !G_local || !eps || !z_hat || !w_hat || !c_local)
    return arg_error("cerot_rows_shard: NULL argument");
  Workspace ws;
  st = check_ws(workspace, ws_bytes, 1, n, m, R, dtype, &ws);
  if (st) return st;
  const IterArgs a = make_args(alpha, nullptr, C_local, G_local, 1, n, m, dtype, eps, 0.0, 1, flags, w_hat,
                               const_cast<double*>(z_hat), row_begin, R);
  cudaStream_t s = (cudaStream_t)stream;
  COT_CHECK_CUDA(rows_pass(a, ws, 0, s));
  COT_CHECK_CUDA(launch_colsum(ws, unit_plan(1, R, device_sm_count()), 1, m, 0, c_local, s));
  return COT_OK;
}

int cerot_zupdate(const double* beta, const double* c, int64_t n, int64_t m, double tol, int64_t check_every,
                  double* z_hat, void* workspace, size_t ws_bytes, void* stream) {
  if (n < 1 || m < 1 || !beta || !c || !z_hat) return arg_error("cerot_zupdate: bad arguments");
  if (tol < 0) return arg_error("cerot_zupdate: tol >= 0 required");
  const size_t need = carve_workspace(nullptr, 1, n, m, 1, COT_F32, device_sm_count(), nullptr);
  if (!workspace || ws_bytes < need) {
    set_error("workspace too small");
    return COT_E_WORKSPACE;
  }
  Workspace ws;   // only the state / counters / monitor offsets are used (they do not depend on R, n, dtype)
  carve_workspace(workspace, 1, n, m, 1, COT_F32, device_sm_count(), &ws);
  COT_CHECK_CUDA(launch_zupdate(c, beta, 1, m, n, tol, check_every, z_hat, ws, (cudaStream_t)stream));
  return COT_OK;
}

int cerot_iter_sharded(const double* alpha, const double* beta, const void* C_local, const void* G_local, int64_t n,
                       int64_t m, int64_t row_begin, int64_t R, int dtype, const double* eps, int64_t iters,
                       double tol, int64_t check_every, uint32_t flags, double* w_hat, double* z_hat, void* workspace,
                       size_t ws_bytes, void* comm, void* stream) {
  int st = check_shape(1, n, m, dtype);
  if (st) return st;
  if (flags & COT_DETERMINISTIC)
    return arg_error("cerot_iter_sharded: COT_DETERMINISTIC is implemented by the persistent kernel only (cerot_iter, "
                     "cerot_iter_fused); the split row pass has no fixed-point partials");
  if (R < 1 || row_begin < 0 || row_begin + R > m) return arg_error("cerot_iter_sharded: bad row range");
  if (!alpha || !beta || !C_local || !G_local || !eps || !w_hat || !z_hat)
    return arg_error("cerot_iter_sharded: NULL argument");
  if (iters < 0 || tol < 0) return arg_error("cerot_iter_sharded: iters >= 0 and tol >= 0 required");
  if (comm && !nccl_api().ok) {
    set_error(nccl_api().err);
    return COT_E_NCCL;
  }
  Workspace ws;
  st = check_ws(workspace, ws_bytes, 1, n, m, R, dtype, &ws);
  if (st) return st;
  const IterArgs a = make_args(alpha, beta, C_local, G_local, 1, n, m, dtype, eps, tol, check_every, flags, w_hat,
                               z_hat, row_begin, R);
  const UnitPlan up = unit_plan(1, R, device_sm_count());
  cudaStream_t s = (cudaStream_t)stream;
  // one iteration t: row pass, rank-local column sums, the exchange, q-update
  auto enqueue = [&](int64_t t, cudaStream_t q) -> int {
    COT_CHECK_CUDA(rows_pass(a, ws, (int)(t & 1), q));
    COT_CHECK_CUDA(launch_colsum(ws, up, 1, m, (int)(t & 1), ws.c_local, q));
    const double* c = ws.c_local;
    if (comm) {   // the exchange step: one m-length fp64 allreduce over NVLink / NVSwitch per iteration
      COT_CHECK_NCCL(nccl_api().AllReduce(ws.c_local, ws.c_global, (size_t)m, ncclFloat64, ncclSum, (ncclComm_t)comm, q));
      c = ws.c_global;
    }
    COT_CHECK_CUDA(launch_zupdate(c, beta, 1, m, n, tol, check_every, z_hat, ws, q));
    return COT_OK;
  };
  // The iteration has no host-side dependence (the freeze rule is applied on the device), so kUnroll iterations
  // (an even count: the row pass alternates its two buffers) are captured ONCE as a CUDA graph, allreduce
  // included, and replayed: one graph launch per kUnroll iterations instead of 3 kernel launches + 1 NCCL call
  // each. Capture is on a private stream (the caller's may be the legacy stream); if it fails (e.g. an NCCL
  // build without capture support) the plain per-iteration enqueue below runs everything.
  constexpr int64_t kUnroll = 8;
  int64_t t0 = 0;
  if (iters >= 2 * kUnroll && !getenv("COT_SHARDED_NO_GRAPH")) {
    cudaStream_t cs = nullptr;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    bool ok = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) == cudaSuccess;
    if (ok) ok = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
      bool body_ok = true;
      for (int64_t t = 0; t < kUnroll && body_ok; ++t) body_ok = enqueue(t, cs) == COT_OK;
      ok = cudaStreamEndCapture(cs, &g) == cudaSuccess && body_ok;
    }
    if (ok) ok = cudaGraphInstantiate(&ge, g, 0) == cudaSuccess;
    if (ok) {
      for (; t0 + kUnroll <= iters; t0 += kUnroll) COT_CHECK_CUDA(cudaGraphLaunch(ge, s));
    } else {
      cudaGetLastError();   // a failed capture leaves nothing enqueued; fall back to the plain loop
      t0 = 0;
    }
    if (ge) cudaGraphExecDestroy(ge);   // freed once the in-flight launches complete
    if (g) cudaGraphDestroy(g);
    if (cs) cudaStreamDestroy(cs);
  }
  for (int64_t t = t0; t < iters; ++t) {
    st = enqueue(t, s);
    if (st) return st;
  }
  return COT_OK;
}

// ------------------------------------------------------------------------------ fused row sharding
size_t cot_xchg_bytes(int64_t m, int nranks) {
  if (m < 1 || nranks < 1 || nranks > kMaxRanks) return 0;
  return cot::xchg_res_offset(m, nranks) + kXchgResHeader + (size_t)3 * m * 8;   // + K-ITER-RES counters and sums
}

int cot_xchg_alloc(int64_t m, int nranks, void** xbuf, void* ipc_handle) {
  const size_t bytes = cot_xchg_bytes(m, nranks);
  if (!bytes || !xbuf) return arg_error("cot_xchg_alloc: need m >= 1, 1 <= nranks <= COT_MAX_RANKS, xbuf");
  void* p = nullptr;
  COT_CHECK_CUDA(cudaMalloc(&p, bytes));
  cudaError_t e = cudaMemset(p, 0, bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess && ipc_handle) {
    cudaIpcMemHandle_t h;
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    e = cudaIpcGetMemHandle(&h, p);
    if (e == cudaSuccess) memcpy(ipc_handle, &h, sizeof(h));
  }
  if (e != cudaSuccess) {
    cudaFree(p);
    set_error(std::string("cot_xchg_alloc: ") + cudaGetErrorString(e));
    return COT_E_CUDA;
  }
  *xbuf = p;
  return COT_OK;
}

int cot_xchg_open(const void* ipc_handle, void** peer_xbuf) {
  if (!ipc_handle || !peer_xbuf) return arg_error("cot_xchg_open: NULL argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  COT_CHECK_CUDA(cudaIpcOpenMemHandle(peer_xbuf, h, cudaIpcMemLazyEnablePeerAccess));
  return COT_OK;
}

int cot_xchg_close(void* peer_xbuf) {
  if (!peer_xbuf) return COT_OK;
  COT_CHECK_CUDA(cudaIpcCloseMemHandle(peer_xbuf));
  return COT_OK;
}

int cot_xchg_free(void* xbuf) {
  if (!xbuf) return COT_OK;
  COT_CHECK_CUDA(cudaFree(xbuf));
  return COT_OK;
}

static int fused_rank_args(const double* alpha, const double* beta, const void* C_local, const void* G_local,
                           int64_t n, int64_t m, int64_t row_begin, int64_t R, int dtype, const double* eps,
                           double tol, int64_t check_every, uint32_t flags, double* w_hat, double* z_hat,
                           void* workspace, size_t ws_bytes, int nranks, int rank, void* const* xbufs,
                           FusedRank* fr) {
  int st = check_shape(1, n, m, dtype);
  if (st) return st;
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks)
    return arg_error("fused sharding: need 1 <= nranks <= COT_MAX_RANKS and 0 <= rank < nranks");
  if (R < 1 || row_begin < 0 || row_begin + R > m) return arg_error("fused sharding: bad row range");
  if (nranks > 1 && R != m / nranks && R != (m + nranks - 1) / nranks)
    return arg_error("fused sharding: R must be floor or ceil of m / nranks (balanced partition)");
  if (!alpha || !beta || !C_local || !G_local || !eps || !w_hat || !z_hat || !xbufs)
    return arg_error("fused sharding: NULL argument");
  for (int q = 0; q < nranks; ++q)
    if (!xbufs[q]) return arg_error("fused sharding: NULL exchange buffer");
  if (tol < 0) return arg_error("fused sharding: tol >= 0 required");
  st = check_ws(workspace, ws_bytes, 1, n, m, R, dtype, &fr->ws);
  if (st) return st;
  fr->a = make_args(alpha, beta, C_local, G_local, 1, n, m, dtype, eps, tol, check_every, flags, w_hat, z_hat,
                    row_begin, R);
  if (!tma_eligible(fr->a))
    return arg_error("fused sharding needs fp32 costs, m % 4 == 0 and m <= 1024 (else cerot_iter_sharded)");
  for (int q = 0; q < kMaxRanks; ++q)
    fr->xpeer[q] = q < nranks ? reinterpret_cast<uint4*>(static_cast<char*>(xbufs[q]) + kXchgHeader) : nullptr;
  fr->xepoch = static_cast<unsigned long long*>(xbufs[rank]);
  fr->rank = rank;
  for (int q = 0; q < kMaxRanks; ++q)
    fr->xres[q] = q < nranks ? static_cast<unsigned char*>(xbufs[q]) + cot::xchg_res_offset(m, nranks) : nullptr;
  return COT_OK;
}

int cerot_iter_fused(const double* alpha, const double* beta, const void* C_local, const void* G_local, int64_t n,
                     int64_t m, int64_t row_begin, int64_t R, int dtype, const double* eps, int64_t iters, double tol,
                     int64_t check_every, uint32_t flags, double* w_hat, double* z_hat, void* workspace,
                     size_t ws_bytes, int nranks, int rank, void* const* xbufs, void* stream) {
  if (iters < 0) return arg_error("cerot_iter_fused: iters >= 0 required");
  FusedRank fr;
  int st = fused_rank_args(alpha, beta, C_local, G_local, n, m, row_begin, R, dtype, eps, tol, check_every, flags,
                           w_hat, z_hat, workspace, ws_bytes, nranks, rank, xbufs, &fr);
  if (st) return st;
  if (iters == 0) return COT_OK;
  if (res_fused_config(fr, nranks, false, nullptr)) {
    COT_CHECK_CUDA(launch_iter_res_fused(&fr, 1, nranks, false, (int)iters, (cudaStream_t)stream));
    return COT_OK;
  }
  COT_CHECK_CUDA(launch_iter_tma_fused(&fr, 1, nranks, false, (int)iters, (cudaStream_t)stream));
  return COT_OK;
}

int cerot_iter_fused_emulated(int nranks, const double* alpha, const double* beta, const void* const* C_local,
                              const void* const* G_local, int64_t n, int64_t m, const int64_t* row_begin,
                              const int64_t* R, int dtype, const double* eps, int64_t iters, double tol,
                              int64_t check_every, uint32_t flags, double* const* w_hat, double* const* z_hat,
                              void* const* workspace, const size_t* ws_bytes, void* const* xbufs, void* stream) {
  if (iters < 0) return arg_error("cerot_iter_fused_emulated: iters >= 0 required");
  if (nranks < 1 || nranks > kMaxRanks) return arg_error("cerot_iter_fused_emulated: 1 <= nranks <= COT_MAX_RANKS");
  if (!C_local || !G_local || !row_begin || !R || !w_hat || !z_hat || !workspace || !ws_bytes || !xbufs)
    return arg_error("cerot_iter_fused_emulated: NULL array");
  FusedRank fr[kMaxRanks];
  for (int v = 0; v < nranks; ++v) {
    int st = fused_rank_args(alpha, beta, C_local[v], G_local[v], n, m, row_begin[v], R[v], dtype, eps, tol,
                             check_every, flags, w_hat[v], z_hat[v], workspace[v], ws_bytes[v], nranks, v, xbufs, &fr[v]);
    if (st) return st;
  }
  if (iters == 0) return COT_OK;
  if (res_fused_config(fr[0], nranks, true, nullptr)) {
    COT_CHECK_CUDA(launch_iter_res_fused(fr, nranks, nranks, true, (int)iters, (cudaStream_t)stream));
    return COT_OK;
  }
  COT_CHECK_CUDA(launch_iter_tma_fused(fr, nranks, nranks, true, (int)iters, (cudaStream_t)stream));
  return COT_OK;
}

int cerot_plan_sharded(const double* alpha, const double* beta, const void* C_local, const void* G_local, int64_t n,
                       int64_t m, int64_t row_begin, int64_t R, int dtype, const double* eps, const double* w_hat,
                       const double* z_hat, void* T_local, double* d_report, void* workspace, size_t ws_bytes,
                       void* comm, void* stream) {
  int st = check_shape(1, n, m, dtype);
  if (st) return st;
  if (R < 1 || row_begin < 0 || row_begin + R > m) return arg_error("cerot_plan_sharded: bad row range");
  if (!alpha || !beta || !C_local || !G_local || !eps || !w_hat || !z_hat)
    return arg_error("cerot_plan_sharded: NULL argument");
  if (comm && !nccl_api().ok) {
    set_error(nccl_api().err);
    return COT_E_NCCL;
  }
  Workspace ws;
  st = check_ws(workspace, ws_bytes, 1, n, m, R, dtype, &ws);
  if (st) return st;
  IterArgs a = make_args(alpha, beta, C_local, G_local, 1, n, m, dtype, eps, 0.0, 1, 0, const_cast<double*>(w_hat),
                         const_cast<double*>(z_hat), row_begin, R);
  return plan_and_report(a, ws, T_local, d_report, comm, (cudaStream_t)stream);
}

// Whole row-sharded solve of this rank (SURVEY §8(b) cerot_solve_sharded): A2 on the held rows, cold start,
// iterations with the NCCL exchange (or none when comm == NULL) and the freeze rule checked every check_every,
// plan of the held rows and the report reduced across ranks.
int cerot_solve_sharded(const double* alpha, const double* beta, const void* C_local, int64_t n, int64_t m,
                        int64_t row_begin, int64_t R, int dtype, const double* eps, double tol, int64_t max_iter,
                        int64_t check_every, uint32_t flags, double* w_hat, double* z_hat, void* T_local,
                        void* workspace, size_t ws_bytes, void* comm, cot_report* report, void* stream) {
  int st = check_shape(1, n, m, dtype);
  if (st) return st;
  if (flags & COT_DETERMINISTIC)
    return arg_error("cerot_solve_sharded: COT_DETERMINISTIC is implemented by the persistent kernel only (cerot_iter, "
                     "cerot_iter_fused); the split row pass has no fixed-point partials");
  if (R < 1 || row_begin < 0 || row_begin + R > m) return arg_error("cerot_solve_sharded: bad row range");
  if (!alpha || !beta || !C_local || !eps || !w_hat || !z_hat || !report)
    return arg_error("cerot_solve_sharded: NULL argument");
  if (max_iter < 0 || tol < 0) return arg_error("cerot_solve_sharded: max_iter >= 0 and tol >= 0 required");
  if (check_every < 1) check_every = 1;
  Workspace ws;
  st = check_ws(workspace, ws_bytes, 1, n, m, R, dtype, &ws);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  COT_CHECK_CUDA(launch_aggregate(C_local, 1, n, m, dtype, ws.G, ws.A, ws.nonfinite, s, R));
  st = cot_check_nonfinite(ws.nonfinite, stream);
  if (st) return st;
  COT_CHECK_CUDA(launch_init(alpha, beta, 1, m, flags | COT_COLD_START, z_hat, ws, s));
  int64_t done = 0, it = 0;
  int32_t conv = 0;
  double res = 0.0;
  while (done < max_iter) {
    const int64_t chunk = std::min<int64_t>(check_every, max_iter - done);
    st = cerot_iter_sharded(alpha, beta, C_local, ws.G, n, m, row_begin, R, dtype, eps, chunk, tol, check_every, flags,
                            w_hat, z_hat, workspace, ws_bytes, comm, stream);
    if (st) return st;
    done += chunk;
    if (tol > 0.0) {
      st = cerot_state(workspace, 1, m, n, dtype, &it, &conv, &res, stream);
      if (st) return st;
      if (conv) break;
    }
  }
  double* d_rep = ws.report;
  st = cerot_plan_sharded(alpha, beta, C_local, ws.G, n, m, row_begin, R, dtype, eps, w_hat, z_hat, T_local, d_rep,
                          workspace, ws_bytes, comm, stream);
  if (st) return st;
  double h[kReportDoubles];
  COT_CHECK_CUDA(cudaMemcpyAsync(h, d_rep, sizeof(h), cudaMemcpyDeviceToHost, s));
  st = cerot_state(workspace, 1, m, n, dtype, &it, &conv, &res, stream);
  if (st) return st;
  report->objective = h[0];
  report->reg_primal = h[1];
  report->dual = h[2];
  report->row_l1 = h[3];
  report->col_l1 = h[4];
  report->col_l2 = h[5];
  report->mass = h[6];
  report->residual = h[7];
  report->iters = it;
  report->converged = conv;
  report->status = (tol > 0.0 && !conv) ? COT_NOT_CONVERGED : COT_OK;
  return report->status;
}

}  // extern "C"
