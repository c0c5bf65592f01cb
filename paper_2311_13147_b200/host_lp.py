"""The small LOT of Theorem 1 (eq. small_problem_CLOT): Alg. 1 line 2, the paper's serial step,
run host-side and outside the hot path (BASELINE.json north_star). The solver is libcyclicot's host C++
primal network simplex (clot_small_lot, NEXT-4; the algorithm the paper names).

clot_solve() chains the device kernels around it: clot_aggregate (GPU) -> G to host -> LP -> S* to device
-> clot_expand (GPU). The LP is the only host computation; nothing here is part of the timed hot path.
"""
from __future__ import annotations

import numpy as np

from . import clot_aggregate, clot_expand


def small_lot(alpha: np.ndarray, beta: np.ndarray, G: np.ndarray, duals: bool = False):
    """min <G, S> s.t. S 1 = alpha, S^T 1 = beta, S >= 0 by the network simplex (clot_small_lot, host C++).
    Returns (value, S) in fp64, plus (u, v, pivots) when duals=True."""
    import ctypes
    from . import _check, lib
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    b = np.ascontiguousarray(beta, dtype=np.float64)
    Gc = np.ascontiguousarray(G, dtype=np.float64)
    m = Gc.shape[0]
    S = np.zeros((m, m))
    u = np.zeros(m)
    v = np.zeros(m)
    val = ctypes.c_double()
    piv = ctypes.c_int64()
    P = lambda x: x.ctypes.data_as(ctypes.c_void_p)
    _check(lib().clot_small_lot(P(a), P(b), P(Gc), m, P(S), ctypes.byref(val), P(u), P(v), ctypes.byref(piv)),
           "clot_small_lot")
    if duals:
        return float(val.value), S, u, v, int(piv.value)
    return float(val.value), S


def clot_solve(C, alpha: np.ndarray, beta: np.ndarray, expand: bool = True, stream=None):
    """Algorithm 1 with lines 1 and 3-6 on the GPU and line 2 on the host.
    C: device tensor [n][m][m]. Returns dict(value = n <G, S*> (full scale), S, G, argmin, T_full)."""
    import torch
    n = C.shape[0]
    import ctypes
    from . import _check, lib
    G, A = clot_aggregate(C, stream=stream)
    Gh = np.ascontiguousarray(G.double().cpu().numpy())
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    b = np.ascontiguousarray(beta, dtype=np.float64)
    m = Gh.shape[0]
    S = np.zeros((m, m))
    full, small = ctypes.c_double(), ctypes.c_double()
    Pn = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _check(lib().clot_lot_value(Pn(a), Pn(b), Pn(Gh), m, n, Pn(S), ctypes.byref(full), ctypes.byref(small)),
           "clot_lot_value")   # the full-scale factor n is applied by the library
    S_dev = torch.as_tensor(S, dtype=C.dtype, device=C.device)   # rounded once to the problem dtype
    T = clot_expand(S_dev, n, argmin=A, stream=stream) if expand else None
    return {"value": full.value, "small_value": small.value, "S": S_dev, "G": G, "argmin": A, "T_full": T}
