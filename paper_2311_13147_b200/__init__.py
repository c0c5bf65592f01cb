"""paper_2311_13147_b200 — B200-native (sm_100a) hot path of "Optimal Transport with Cyclic Symmetry"
(arXiv 2311.13147): C-LOT aggregation, cyclic Sinkhorn (C-EROT) iterations, plan reconstruction and the
d x d block-circulant expansion, behind the C ABI of include/cyclicot.h (libcyclicot.so).

This module is a thin ctypes binding: it marshals torch tensors (device memory, streams) into the C ABI
and raises on error codes. Every step of the path runs in the library's CUDA kernels; there is no CPU
fallback — if libcyclicot.so is missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcyclicot.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "cyclicot.h")

COT_F32, COT_F64 = 0, 1
COT_COLD_START, COT_FORCE_LDG, COT_PRECOMPUTED, COT_FORCE_TMA, COT_DETERMINISTIC = 0x1, 0x2, 0x4, 0x8, 0x10
STATUS = {0: "COT_OK", 1: "COT_NOT_CONVERGED", -1: "COT_E_ARG", -2: "COT_E_NONFINITE", -3: "COT_E_MARGINAL",
          -4: "COT_E_CUDA", -5: "COT_E_NCCL", -6: "COT_E_WORKSPACE", -7: "COT_E_UNDERFLOW", -8: "COT_E_PEER"}
REPORT_FIELDS = ("objective", "reg_primal", "dual", "row_l1", "col_l1", "col_l2", "mass", "residual")


class CotError(RuntimeError):
    def __init__(self, code: int, fn: str, msg: str):
        super().__init__(f"{fn}: {STATUS.get(code, code)}: {msg}")
        self.code = code


class cot_report(ctypes.Structure):
    _fields_ = [(f, ctypes.c_double) for f in REPORT_FIELDS] + [
        ("iters", ctypes.c_int64), ("converged", ctypes.c_int32), ("status", ctypes.c_int32)]


_lib = None
_vp, _i64, _i32, _u32, _dbl, _sz = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32,
                                    ctypes.c_double, ctypes.c_size_t)

_SIGS = {
    "cot_abi_version": (ctypes.c_int, []),
    "cot_last_error": (ctypes.c_char_p, []),
    "cot_workspace_bytes": (_sz, [_i64, _i64, _i64, ctypes.c_int]),
    "clot_aggregate": (ctypes.c_int, [_vp, _i64, _i64, _i64, ctypes.c_int, _vp, _vp, _vp, _vp]),
    "cot_check_nonfinite": (ctypes.c_int, [_vp, _vp]),
    "clot_expand": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i64, ctypes.c_int, _vp, _vp]),
    "cerot_init": (ctypes.c_int, [_vp, _vp, _i64, _i64, _u32, _vp, _vp, _sz, _vp]),
    "cot_iter_path": (ctypes.c_int, [_i64, _i64, _i64, ctypes.c_int, _u32]),
    "cot_fused_path": (ctypes.c_int, [_i64, _i64, _i64, ctypes.c_int, ctypes.c_int, _u32]),
    "cot_expand_path": (ctypes.c_int, [_i64, _i64, ctypes.c_int]),
    "cot_set_device": (ctypes.c_int, [ctypes.c_int]),
    "cerot_iter": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, ctypes.c_int, _vp, _i64, _dbl, _i64, _u32,
                                  _vp, _vp, _vp, _sz, _vp]),
    "cerot_rows": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, ctypes.c_int, _vp, _u32, _vp, _vp, _vp, _sz,
                                  ctypes.c_int, _vp]),
    "cerot_cols": (ctypes.c_int, [_vp, _i64, _i64, _i64, ctypes.c_int, _dbl, _i64, _vp, _vp, _sz, ctypes.c_int, _vp]),
    "cerot_state": (ctypes.c_int, [_vp, _i64, _i64, _i64, ctypes.c_int, _vp, _vp, _vp, _vp]),
    "cerot_plan": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp,
                                  _sz, _vp]),
    "cerot_solve": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, ctypes.c_int, _vp, _dbl, _i64, _i64, _u32, _vp,
                                   _vp, _vp, _vp, _sz, ctypes.POINTER(cot_report), _vp]),
    "csrot_solve": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, ctypes.c_int, ctypes.c_int, _vp, _dbl, _i64, _i64,
                                   _u32, _vp, _vp, _vp, _vp, _sz, ctypes.POINTER(cot_report), _vp]),
    "cerot_precompute": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i64, ctypes.c_int, _vp, _vp, _vp]),
    # row sharding (dist.py)
    "cot_workspace_bytes_sharded": (_sz, [_i64, _i64, _i64, ctypes.c_int]),
    "clot_aggregate_shard": (ctypes.c_int, [_vp, _i64, _i64, _i64, ctypes.c_int, _vp, _vp, _vp, _vp]),
    "clot_expand_shard": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i64, ctypes.c_int, _vp, _vp]),
    "cot_nccl_unique_id": (ctypes.c_int, [_vp]),
    "cot_comm_init": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "cot_comm_destroy": (ctypes.c_int, [_vp]),
    "cerot_rows_shard": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, _i64, ctypes.c_int, _vp, _u32, _vp, _vp, _vp,
                                        _vp, _sz, _vp]),
    "cerot_zupdate": (ctypes.c_int, [_vp, _vp, _i64, _i64, _dbl, _i64, _vp, _vp, _sz, _vp]),
    "cerot_iter_sharded": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, ctypes.c_int, _vp, _i64, _dbl,
                                          _i64, _u32, _vp, _vp, _vp, _sz, _vp, _vp]),
    "cerot_plan_sharded": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, ctypes.c_int, _vp, _vp, _vp,
                                          _vp, _vp, _vp, _sz, _vp, _vp]),
    # NEXT-2: two-stage Sinkhorn (Alg. 3)
    "cot_two_stage_workspace_bytes": (_sz, [_i64, _i64, ctypes.c_int]),
    "cerot_two_stage": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, ctypes.c_int, _vp, _i64, _dbl, _i64, _dbl, _i64,
                                       _vp, _vp, _vp, _vp, _vp, _sz, ctypes.POINTER(cot_report),
                                       ctypes.POINTER(_i64), _vp]),
    "cerot_two_stage_gap": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, ctypes.c_int, _vp, _i64, _dbl, _i64, _dbl,
                                           _dbl, _i64, _vp, _vp, _vp, _vp, _vp, _sz, ctypes.POINTER(cot_report),
                                           ctypes.POINTER(_i64), _vp]),
    # NEXT-4: host network simplex for the small LOT (host pointers)
    "clot_small_lot": (ctypes.c_int, [_vp, _vp, _vp, _i64, _vp, ctypes.POINTER(_dbl), _vp, _vp,
                                      ctypes.POINTER(_i64)]),
    "clot_lot_value": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _vp, ctypes.POINTER(_dbl), ctypes.POINTER(_dbl)]),
    "cerot_solve_sharded": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, _i64, ctypes.c_int, _vp, _dbl, _i64,
                                           _i64, _u32, _vp, _vp, _vp, _vp, _sz, _vp, ctypes.POINTER(cot_report),
                                           _vp]),
    # fused row sharding (in-kernel peer exchange; dist.py)
    "cot_xchg_bytes": (_sz, [_i64, ctypes.c_int]),
    "cot_xchg_alloc": (ctypes.c_int, [_i64, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p), _vp]),
    "cot_xchg_open": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_void_p)]),
    "cot_xchg_close": (ctypes.c_int, [_vp]),
    "cot_xchg_free": (ctypes.c_int, [_vp]),
    "cot_xchg_nccl_alloc": (ctypes.c_int, [_vp, _i64, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                                           ctypes.POINTER(ctypes.c_void_p)]),
    "cot_xchg_nccl_peers": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "cot_xchg_nccl_free": (ctypes.c_int, [_vp, _vp, _vp]),
    "cerot_iter_fused": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, ctypes.c_int, _vp, _i64, _dbl,
                                        _i64, _u32, _vp, _vp, _vp, _sz, ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_void_p), _vp]),
    "cerot_iter_fused_emulated": (ctypes.c_int, [ctypes.c_int, _vp, _vp, ctypes.POINTER(ctypes.c_void_p),
                                                 ctypes.POINTER(ctypes.c_void_p), _i64, _i64, ctypes.POINTER(_i64),
                                                 ctypes.POINTER(_i64), ctypes.c_int, _vp, _i64, _dbl, _i64, _u32,
                                                 ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p),
                                                 ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(_sz),
                                                 ctypes.POINTER(ctypes.c_void_p), _vp]),
}


def lib():
    """Load libcyclicot.so (built in-tree by __graft_entry__.build()). Raises if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def use_current_device():
    """Point the library's (static) CUDA runtime at torch's current device (one call per process/thread that
    drives a GPU other than device 0; bench.py and dist.py call it after torch.cuda.set_device)."""
    import torch
    _check(lib().cot_set_device(torch.cuda.current_device()), "cot_set_device")


def _check(code: int, fn: str, ok=(0,)):
    if code not in ok:
        raise CotError(code, fn, lib().cot_last_error().decode())
    return code


def _dtype_code(t) -> int:
    import torch
    if t.dtype == torch.float32:
        return COT_F32
    if t.dtype == torch.float64:
        return COT_F64
    raise TypeError(f"cost dtype must be float32 or float64, got {t.dtype}")


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("tensor must live in CUDA device memory")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return t.data_ptr()


def _stream(stream) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _shape(C):
    """(B, n, m, batched) from C [n][m][m] or [B][n][m][m]."""
    if C.dim() == 3:
        return 1, C.shape[0], C.shape[1], False
    if C.dim() == 4:
        return C.shape[0], C.shape[1], C.shape[2], True
    raise ValueError("C must be [n][m][m] or [B][n][m][m]")


# ------------------------------------------------------------------------------------ C-LOT
def clot_aggregate(C, G=None, argmin=None, nonfinite=None, stream=None, check=True):
    """G = min_k C_k and the smallest argmin. Returns (G, argmin)."""
    import torch
    B, n, m, batched = _shape(C)
    shp = (B, m, m) if batched else (m, m)
    G = torch.empty(shp, dtype=C.dtype, device=C.device) if G is None else G
    argmin = torch.empty(shp, dtype=torch.int32, device=C.device) if argmin is None else argmin
    if check and nonfinite is None:
        nonfinite = torch.zeros(1, dtype=torch.int32, device=C.device)
    s = _stream(stream)
    _check(lib().clot_aggregate(_ptr(C), B, n, m, _dtype_code(C), _ptr(G), _ptr(argmin), _ptr(nonfinite), s),
           "clot_aggregate")
    if check:
        _check(lib().cot_check_nonfinite(_ptr(nonfinite), s), "clot_aggregate")
    return G, argmin


def clot_expand(S, n: int, argmin=None, out=None, stream=None):
    """Dense d x d block-circulant plan (Lemma 1). With argmin: S is the small LOT solution
    [.., m, m] lifted by eq. optimal_solution_problem_CLOT; without: S is the n blocks [.., n, m, m]."""
    import torch
    if argmin is not None:
        batched = S.dim() == 3
        B = S.shape[0] if batched else 1
        m = S.shape[-1]
    else:
        batched = S.dim() == 4
        B = S.shape[0] if batched else 1
        m = S.shape[-1]
        assert S.shape[-3] == n
    d = n * m
    shp = (B, d, d) if batched else (d, d)
    out = torch.empty(shp, dtype=S.dtype, device=S.device) if out is None else out
    _check(lib().clot_expand(_ptr(S), _ptr(argmin), B, n, m, _dtype_code(S), _ptr(out), _stream(stream)),
           "clot_expand")
    return out


# ------------------------------------------------------------------------------------ C-EROT
def workspace(B: int, n: int, m: int, dtype_code: int, device="cuda"):
    import torch
    nbytes = int(lib().cot_workspace_bytes(B, n, m, dtype_code))
    return torch.empty(nbytes, dtype=torch.uint8, device=device)


class CerotProblem:
    """Device-resident problem + state for step-by-step use of cerot_init / cerot_iter / cerot_plan.
    Tensors: C [n,m,m] or [B,n,m,m] (fp32/fp64), alpha/beta [.., m] fp64, eps [B] fp64."""

    def __init__(self, C, alpha, beta, eps, stream=None):
        import torch
        self.C = C
        self.B, self.n, self.m, self.batched = _shape(C)
        self.dt = _dtype_code(C)
        self.alpha = alpha.to(torch.float64).contiguous()
        self.beta = beta.to(torch.float64).contiguous()
        self.eps = torch.as_tensor(eps, dtype=torch.float64, device=C.device).reshape(self.B).contiguous()
        self.w_hat = torch.zeros_like(self.alpha)
        self.z_hat = torch.zeros_like(self.beta)
        self.ws = workspace(self.B, self.n, self.m, self.dt, C.device)
        self.stream = stream
        self.G, self.argmin = clot_aggregate(C, stream=stream)

    def init(self, cold: bool = True):
        _check(lib().cerot_init(_ptr(self.alpha), _ptr(self.beta), self.B, self.m, COT_COLD_START if cold else 0,
                                _ptr(self.z_hat), _ptr(self.ws), self.ws.numel(), _stream(self.stream)), "cerot_init")
        return self

    def iterate(self, iters: int, tol: float = 0.0, check_every: int = 1, flags: int = 0):
        _check(lib().cerot_iter(_ptr(self.alpha), _ptr(self.beta), _ptr(self.C), _ptr(self.G), self.B, self.n,
                                self.m, self.dt, _ptr(self.eps), iters, tol, check_every, flags, _ptr(self.w_hat),
                                _ptr(self.z_hat), _ptr(self.ws), self.ws.numel(), _stream(self.stream)), "cerot_iter")
        return self

    # ---- NEXT-1: Alg. 2 with the cyclic Gibbs kernel precomputed, O(m^2) per iteration
    def precompute(self):
        """S_ij = sum_k exp((G_ij - C_ijk)/eps) (cerot_precompute), kept on the device."""
        import torch
        shp = (self.B, 1, self.m, self.m) if self.batched else (1, self.m, self.m)
        self.S = torch.empty(shp, dtype=self.C.dtype, device=self.C.device)
        _check(lib().cerot_precompute(_ptr(self.C), _ptr(self.G), self.B, self.n, self.m, self.dt, _ptr(self.eps),
                                      _ptr(self.S), _stream(self.stream)), "cerot_precompute")
        return self

    def iterate_precomputed(self, iters: int, tol: float = 0.0, check_every: int = 1, flags: int = 0):
        if getattr(self, "S", None) is None:
            self.precompute()
        _check(lib().cerot_iter(_ptr(self.alpha), _ptr(self.beta), _ptr(self.S), _ptr(self.G), self.B, 1, self.m,
                                self.dt, _ptr(self.eps), iters, tol, check_every, flags | COT_PRECOMPUTED,
                                _ptr(self.w_hat), _ptr(self.z_hat), _ptr(self.ws), self.ws.numel(),
                                _stream(self.stream)), "cerot_iter")
        return self

    def rows(self, parity: int, flags: int = 0):
        """The p-update pass alone (cerot_rows)."""
        _check(lib().cerot_rows(_ptr(self.alpha), _ptr(self.C), _ptr(self.G), self.B, self.n, self.m, self.dt,
                                _ptr(self.eps), flags, _ptr(self.z_hat), _ptr(self.w_hat), _ptr(self.ws),
                                self.ws.numel(), parity, _stream(self.stream)), "cerot_rows")

    def cols(self, parity: int, tol: float = 0.0, check_every: int = 1):
        """The column reduction + q-update alone (cerot_cols)."""
        _check(lib().cerot_cols(_ptr(self.beta), self.B, self.n, self.m, self.dt, tol, check_every, _ptr(self.z_hat),
                                _ptr(self.ws), self.ws.numel(), parity, _stream(self.stream)), "cerot_cols")

    def state(self):
        it = (ctypes.c_int64 * self.B)()
        cv = (ctypes.c_int32 * self.B)()
        rs = (ctypes.c_double * self.B)()
        _check(lib().cerot_state(_ptr(self.ws), self.B, self.m, self.n, self.dt, it, cv, rs, _stream(self.stream)),
               "cerot_state")
        return np.array(it[:]), np.array(cv[:]), np.array(rs[:])

    def plan(self, T_blocks: bool = False, report=None):
        import torch
        T = torch.empty_like(self.C) if T_blocks else None
        rep = torch.empty((self.B, 8), dtype=torch.float64, device=self.C.device) if report is None else report
        _check(lib().cerot_plan(_ptr(self.alpha), _ptr(self.beta), _ptr(self.C), _ptr(self.G), self.B, self.n,
                                self.m, self.dt, _ptr(self.eps), _ptr(self.w_hat), _ptr(self.z_hat), _ptr(T),
                                _ptr(rep), _ptr(self.ws), self.ws.numel(), _stream(self.stream)), "cerot_plan")
        return T, rep


def report_dict(rep_row) -> dict:
    v = [float(x) for x in rep_row]
    return dict(zip(REPORT_FIELDS, v))


def cerot_solve(C, alpha, beta, eps, tol=0.0, max_iter=1000, check_every=1, T_blocks=False, cold=True,
                w_hat=None, z_hat=None, ws=None, stream=None):
    """Whole C-EROT solve on the device (A2..A5). Returns (w_hat, z_hat, T_blocks or None, [report dict])."""
    import torch
    B, n, m, batched = _shape(C)
    dt = _dtype_code(C)
    alpha = alpha.to(torch.float64).contiguous()
    beta = beta.to(torch.float64).contiguous()
    eps_t = torch.as_tensor(eps, dtype=torch.float64, device=C.device).reshape(B).contiguous()
    w_hat = torch.zeros_like(alpha) if w_hat is None else w_hat
    z_hat = torch.zeros_like(beta) if z_hat is None else z_hat
    ws = workspace(B, n, m, dt, C.device) if ws is None else ws
    T = torch.empty_like(C) if T_blocks else None
    reps = (cot_report * B)()
    code = lib().cerot_solve(_ptr(alpha), _ptr(beta), _ptr(C), B, n, m, dt, _ptr(eps_t), tol, max_iter, check_every,
                             COT_COLD_START if cold else 0, _ptr(w_hat), _ptr(z_hat), _ptr(T), _ptr(ws), ws.numel(),
                             reps, _stream(stream))
    _check(code, "cerot_solve", ok=(0, 1))
    out = []
    for r in reps:
        d = {f: getattr(r, f) for f in REPORT_FIELDS}
        d.update(iters=r.iters, converged=bool(r.converged), status=STATUS[r.status])
        out.append(d)
    return w_hat, z_hat, T, out


COT_REG_SQUARED = 1


def csrot_solve(C, alpha, beta, gamma, tol=0.0, max_sweeps=1000, check_every=1, T_blocks=False, stream=None):
    """NEXT-3: C-SROT with the squared regulariser on the device. Returns (w, z, T or None,
    [report dict]); w, z in cost units."""
    import torch
    B, n, m, batched = _shape(C)
    dt = _dtype_code(C)
    alpha = alpha.to(torch.float64).contiguous()
    beta = beta.to(torch.float64).contiguous()
    gam = torch.as_tensor(gamma, dtype=torch.float64, device=C.device).reshape(-1).expand(B).contiguous()
    w = torch.zeros_like(alpha)
    z = torch.zeros_like(beta)
    ws = workspace(B, n, m, dt, C.device)
    T = torch.empty_like(C) if T_blocks else None
    reps = (cot_report * B)()
    code = lib().csrot_solve(_ptr(alpha), _ptr(beta), _ptr(C), B, n, m, dt, COT_REG_SQUARED, _ptr(gam), tol,
                             max_sweeps, check_every, COT_COLD_START, _ptr(w), _ptr(z), _ptr(T), _ptr(ws), ws.numel(),
                             reps, _stream(stream))
    _check(code, "csrot_solve", ok=(0, 1))
    out = []
    for r in reps:
        d = {f: getattr(r, f) for f in REPORT_FIELDS}
        d.update(iters=r.iters, converged=bool(r.converged), status=STATUS[r.status])
        out.append(d)
    return w, z, T, out


def two_stage_sinkhorn(a, b, C, eps, iters1, iters2, tol1=0.0, tol2=0.0, check_every=1, stream=None,
                       obj_ref=None, tol_obj=0.0):
    """NEXT-2: Algorithm 3 on the device (cerot_two_stage). a, b: device [d] fp64 (approximately
    n-periodic), C: device [n][m][m]. Returns (f_hat, g_hat [d], w_hat, z_hat [m], report dict) with
    eps-scaled potentials; report values are full-problem (no factor n). With obj_ref and tol_obj > 0 stage 2
    stops on App. F's objective gap instead of tol2 (cerot_two_stage_gap)."""
    import torch
    n, m = C.shape[0], C.shape[1]
    dt = _dtype_code(C)
    dev = C.device
    a = a.to(torch.float64).contiguous()
    b = b.to(torch.float64).contiguous()
    eps_t = torch.as_tensor(eps, dtype=torch.float64, device=dev).reshape(1).contiguous()
    f = torch.zeros(n * m, dtype=torch.float64, device=dev)
    g = torch.zeros_like(f)
    w = torch.zeros(m, dtype=torch.float64, device=dev)
    z = torch.zeros_like(w)
    ws = torch.empty(int(lib().cot_two_stage_workspace_bytes(n, m, dt)), dtype=torch.uint8, device=dev)
    rep = cot_report()
    its = (ctypes.c_int64 * 2)()
    if obj_ref is not None:
        code = lib().cerot_two_stage_gap(_ptr(a), _ptr(b), _ptr(C), n, m, dt, _ptr(eps_t), iters1, tol1, iters2,
                                         float(obj_ref), float(tol_obj), check_every, _ptr(f), _ptr(g), _ptr(w),
                                         _ptr(z), _ptr(ws), ws.numel(), ctypes.byref(rep), its, _stream(stream))
    else:
        code = lib().cerot_two_stage(_ptr(a), _ptr(b), _ptr(C), n, m, dt, _ptr(eps_t), iters1, tol1, iters2, tol2,
                                     check_every, _ptr(f), _ptr(g), _ptr(w), _ptr(z), _ptr(ws), ws.numel(),
                                     ctypes.byref(rep), its, _stream(stream))
    _check(code, "cerot_two_stage", ok=(0, 1))
    d = {k: getattr(rep, k) for k in REPORT_FIELDS}
    d.update(iters1=int(its[0]), iters2=int(its[1]), converged=bool(rep.converged), status=STATUS[rep.status])
    return f, g, w, z, d
