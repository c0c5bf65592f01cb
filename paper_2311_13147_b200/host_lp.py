"""The small LOT of Theorem 1 (eq. small_problem_CLOT): Alg. 1 line 2, the paper's serial step,
run host-side and outside the hot path (BASELINE.json north_star). HiGHS (scipy) is the LP library used.

clot_solve() chains the device kernels around it: clot_aggregate (GPU) -> G to host -> LP -> S* to device
-> clot_expand (GPU). The LP is the only host computation; nothing here is part of the timed hot path.
"""
from __future__ import annotations

import numpy as np
import scipy.optimize
import scipy.sparse

from . import clot_aggregate, clot_expand


def small_lot(alpha: np.ndarray, beta: np.ndarray, G: np.ndarray):
    """min <G, S> s.t. S 1 = alpha, S^T 1 = beta, S >= 0 (HiGHS). Returns (value, S) in fp64."""
    m = G.shape[0]
    rows = scipy.sparse.kron(scipy.sparse.eye(m), np.ones((1, m)))
    cols = scipy.sparse.kron(np.ones((1, m)), scipy.sparse.eye(m))
    A_eq = scipy.sparse.vstack([rows, cols]).tocsr()
    res = scipy.optimize.linprog(np.asarray(G, np.float64).ravel(), A_eq=A_eq,
                                 b_eq=np.concatenate([alpha, beta]), bounds=(0, None), method="highs")
    if res.status != 0:
        raise RuntimeError(f"small LOT failed: {res.message}")
    S = np.maximum(res.x.reshape(m, m), 0.0)
    return float(np.asarray(G, np.float64).ravel() @ res.x), S


def clot_solve(C, alpha: np.ndarray, beta: np.ndarray, expand: bool = True, stream=None):
    """Algorithm 1 with lines 1 and 3-6 on the GPU and line 2 on the host.
    C: device tensor [n][m][m]. Returns dict(value = n <G, S*> (full scale), S, G, argmin, T_full)."""
    import torch
    n = C.shape[0]
    G, A = clot_aggregate(C, stream=stream)
    Gh = G.double().cpu().numpy()
    small, S = small_lot(np.asarray(alpha, np.float64), np.asarray(beta, np.float64), Gh)
    S_dev = torch.as_tensor(S, dtype=C.dtype, device=C.device)   # rounded once to the problem dtype
    T = clot_expand(S_dev, n, argmin=A, stream=stream) if expand else None
    return {"value": n * small, "small_value": small, "S": S_dev, "G": G, "argmin": A, "T_full": T}
