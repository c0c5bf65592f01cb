// C ABI of libcyclicot (include/cyclicot.h): argument validation, workspace carving, launch sequencing.
// No compute happens here: every step of the path is one of the kernels in k_*.cu.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <cmath>
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

size_t carve_workspace(void* base, int64_t B, int64_t n, int64_t m, int dtype, int sm_count, Workspace* ws) {
  (void)n;
  const UnitPlan up = unit_plan(B, m, sm_count);
  const size_t esz = dtype == COT_F32 ? 4 : 8;
  const int64_t ntiles = (m + 31) / 32;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 256);
    return base ? static_cast<char*>(base) + o : nullptr;
  };
  // Order matters: the per-problem state comes first so its offset depends on B only (cerot_init and
  // cerot_state find it without knowing n or the dtype); the dtype-sized G comes last.
  Workspace w{};
  w.state = reinterpret_cast<SolverState*>(take((size_t)B * sizeof(SolverState)));
  w.counters = reinterpret_cast<unsigned*>(take((size_t)B * 4));
  w.grid_bar = reinterpret_cast<unsigned*>(take(16));
  w.nonfinite = reinterpret_cast<int32_t*>(take(4));
  w.report = reinterpret_cast<double*>(take((size_t)B * kReportDoubles * 8));
  w.resid_part = reinterpret_cast<double*>(take((size_t)(B * ntiles) * 8));
  w.plan_scal = reinterpret_cast<double*>(take((size_t)up.U * kPlanScalars * 8));
  w.partials[0] = reinterpret_cast<double*>(take((size_t)(up.U * m) * 8));
  w.partials[1] = reinterpret_cast<double*>(take((size_t)(up.U * m) * 8));
  w.A = reinterpret_cast<int32_t*>(take((size_t)(B * m * m) * 4));
  w.G = take((size_t)(B * m * m) * esz);
  if (ws) *ws = w;
  return off;
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

static int check_ws(void* workspace, size_t ws_bytes, int64_t B, int64_t n, int64_t m, int dtype, Workspace* ws) {
  const size_t need = carve_workspace(nullptr, B, n, m, dtype, device_sm_count(), nullptr);
  if (!workspace || ws_bytes < need) {
    set_error("workspace too small: need " + std::to_string(need) + " bytes, got " + std::to_string(ws_bytes));
    return COT_E_WORKSPACE;
  }
  if (reinterpret_cast<uintptr_t>(workspace) % 256 != 0) {
    set_error("workspace must be 256-byte aligned");
    return COT_E_WORKSPACE;
  }
  carve_workspace(workspace, B, n, m, dtype, device_sm_count(), ws);
  return COT_OK;
}

extern "C" {

int cot_abi_version(void) { return COT_ABI_VERSION; }

const char* cot_last_error(void) { return g_last_error.c_str(); }

size_t cot_workspace_bytes(int64_t B, int64_t n, int64_t m, int dtype) {
  if (B < 1 || n < 1 || m < 1) return 0;
  return carve_workspace(nullptr, B, n, m, dtype, device_sm_count(), nullptr);
}

int clot_aggregate(const void* C, int64_t B, int64_t n, int64_t m, int dtype, void* G, int32_t* argmin,
                   int32_t* d_nonfinite, void* stream) {
  int st = check_shape(B, n, m, dtype);
  if (st) return st;
  if (!C || !G || !argmin) return arg_error("clot_aggregate: C, G and argmin must be non-NULL");
  COT_CHECK_CUDA(launch_aggregate(C, B, n, m, dtype, G, argmin, d_nonfinite, (cudaStream_t)stream));
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
  // the state block is at the start of the workspace for every (n, dtype) (see carve_workspace)
  Workspace ws;
  const size_t need = (size_t)B * (sizeof(SolverState) + 4) + 2048;
  if (!workspace || ws_bytes < need) {
    set_error("workspace too small");
    return COT_E_WORKSPACE;
  }
  carve_workspace(workspace, B, 1, m, COT_F32, device_sm_count(), &ws);
  COT_CHECK_CUDA(launch_init(alpha, beta, B, m, flags, z_hat, ws, (cudaStream_t)stream));
  return COT_OK;
}

static IterArgs make_args(const double* alpha, const double* beta, const void* C, const void* G, int64_t B, int64_t n,
                          int64_t m, int dtype, const double* eps, double tol, int64_t check_every, uint32_t flags,
                          double* w_hat, double* z_hat) {
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
  a.R = m;
  a.row_begin = 0;
  a.dtype = dtype;
  a.tol = tol;
  a.check_every = check_every > 0 ? check_every : 1;
  a.flags = flags;
  return a;
}

int cerot_iter(const double* alpha, const double* beta, const void* C, const void* G, int64_t B, int64_t n, int64_t m,
               int dtype, const double* eps, int64_t iters, double tol, int64_t check_every, uint32_t flags,
               double* w_hat, double* z_hat, void* workspace, size_t ws_bytes, void* stream) {
  int st = check_shape(B, n, m, dtype);
  if (st) return st;
  if (!alpha || !beta || !C || !G || !eps || !w_hat || !z_hat) return arg_error("cerot_iter: NULL argument");
  if (iters < 0 || tol < 0 || !(tol == tol)) return arg_error("cerot_iter: iters >= 0 and tol >= 0 required");
  // the state lives in the same place for every (n, dtype): carve with the caller's shape
  Workspace ws;
  st = check_ws(workspace, ws_bytes, B, n, m, dtype, &ws);
  if (st) return st;
  const IterArgs a = make_args(alpha, beta, C, G, B, n, m, dtype, eps, tol, check_every, flags, w_hat, z_hat);
  const UnitPlan up = unit_plan(B, m, device_sm_count());
  cudaStream_t s = (cudaStream_t)stream;
  if (iters > 0 && tma_eligible(a)) {
    COT_CHECK_CUDA(launch_iter_tma(a, ws, (int)iters, false, 0, s));
    return COT_OK;
  }
  for (int64_t t = 0; t < iters; ++t) {
    COT_CHECK_CUDA(launch_rows(a, ws, up, (int)(t & 1), s));
    COT_CHECK_CUDA(launch_cols(a, ws, up, (int)(t & 1), s));
  }
  return COT_OK;
}

int cerot_rows(const double* alpha, const void* C, const void* G, int64_t B, int64_t n, int64_t m, int dtype,
               const double* eps, uint32_t flags, const double* z_hat, double* w_hat, void* workspace,
               size_t ws_bytes, int parity, void* stream) {
  int st = check_shape(B, n, m, dtype);
  if (st) return st;
  if (!alpha || !C || !G || !eps || !w_hat || !z_hat) return arg_error("cerot_rows: NULL argument");
  Workspace ws;
  st = check_ws(workspace, ws_bytes, B, n, m, dtype, &ws);
  if (st) return st;
  const IterArgs a = make_args(alpha, nullptr, C, G, B, n, m, dtype, eps, 0.0, 1, flags, w_hat,
                               const_cast<double*>(z_hat));
  if (tma_eligible(a)) {
    COT_CHECK_CUDA(launch_iter_tma(a, ws, 1, true, parity & 1, (cudaStream_t)stream));
    return COT_OK;
  }
  COT_CHECK_CUDA(launch_rows(a, ws, unit_plan(B, m, device_sm_count()), parity & 1, (cudaStream_t)stream));
  return COT_OK;
}

int cerot_cols(const double* beta, int64_t B, int64_t n, int64_t m, int dtype, double tol, int64_t check_every,
               double* z_hat, void* workspace, size_t ws_bytes, int parity, void* stream) {
  int st = check_shape(B, n, m, dtype);
  if (st) return st;
  if (!beta || !z_hat) return arg_error("cerot_cols: NULL argument");
  if (tol < 0) return arg_error("cerot_cols: tol >= 0 required");
  Workspace ws;
  st = check_ws(workspace, ws_bytes, B, n, m, dtype, &ws);
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
  carve_workspace(const_cast<void*>(workspace), B, n, m, dtype, device_sm_count(), &ws);
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
  return COT_OK;
}

int cerot_plan(const double* alpha, const double* beta, const void* C, const void* G, int64_t B, int64_t n, int64_t m,
               int dtype, const double* eps, const double* w_hat, const double* z_hat, void* T_blocks,
               double* d_report, void* workspace, size_t ws_bytes, void* stream) {
  int st = check_shape(B, n, m, dtype);
  if (st) return st;
  if (!alpha || !beta || !C || !G || !eps || !w_hat || !z_hat) return arg_error("cerot_plan: NULL argument");
  Workspace ws;
  st = check_ws(workspace, ws_bytes, B, n, m, dtype, &ws);
  if (st) return st;
  IterArgs a = make_args(alpha, beta, C, G, B, n, m, dtype, eps, 0.0, 1, 0, const_cast<double*>(w_hat),
                         const_cast<double*>(z_hat));
  const UnitPlan up = unit_plan(B, m, device_sm_count());
  COT_CHECK_CUDA(launch_plan(a, ws, up, T_blocks, d_report, (cudaStream_t)stream));
  return COT_OK;
}

int cerot_solve(const double* alpha, const double* beta, const void* C, int64_t B, int64_t n, int64_t m, int dtype,
                const double* eps, double tol, int64_t max_iter, int64_t check_every, uint32_t flags, double* w_hat,
                double* z_hat, void* T_blocks, void* workspace, size_t ws_bytes, cot_report* report, void* stream) {
  int st = check_shape(B, n, m, dtype);
  if (st) return st;
  if (!alpha || !beta || !C || !eps || !w_hat || !z_hat || !report) return arg_error("cerot_solve: NULL argument");
  if (max_iter < 0 || tol < 0) return arg_error("cerot_solve: max_iter >= 0 and tol >= 0 required");
  Workspace ws;
  st = check_ws(workspace, ws_bytes, B, n, m, dtype, &ws);
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
  int64_t done = 0;
  while (done < max_iter) {
    const int64_t chunk = std::min<int64_t>(check_every, max_iter - done);
    if (tma_eligible(a)) {
      COT_CHECK_CUDA(launch_iter_tma(a, ws, (int)chunk, false, 0, s));
    } else {
      for (int64_t t = 0; t < chunk; ++t) {
        COT_CHECK_CUDA(launch_rows(a, ws, up, (int)((done + t) & 1), s));
        COT_CHECK_CUDA(launch_cols(a, ws, up, (int)((done + t) & 1), s));
      }
    }
    done += chunk;
    if (tol > 0.0 || done >= max_iter) {
      st = cerot_state(workspace, B, m, n, dtype, it.data(), conv.data(), res.data(), stream);
      if (st) return st;
      bool all = tol > 0.0;
      for (int64_t b = 0; b < B && all; ++b) all = conv[(size_t)b] != 0;
      if (all) break;
    }
  }
  COT_CHECK_CUDA(launch_plan(a, ws, up, T_blocks, ws.report, s));
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

}  // extern "C"
