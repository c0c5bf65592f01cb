"""TEST INFRASTRUCTURE (oracle) — linear OT: the plain LP definition and Algorithm 1 (Fast C-LOT).
HiGHS (scipy.optimize.linprog) is the library LP primitive. See oracle/__init__.py for import rules."""
from __future__ import annotations

import numpy as np
import scipy.optimize
import scipy.sparse

from .core import aggregate, expand_cost, expand_vector, lift

__all__ = ["lot", "clot", "naive_tile_lot", "lot_full"]


def lot(a: np.ndarray, b: np.ndarray, C: np.ndarray):
    """LOT (eq. problem_ROT with the regulariser of eq. reg_for_original_OT):
    min <C, T> s.t. T 1 = a, T^T 1 = b, T >= 0, solved as a plain LP with HiGHS.
    Returns (value, T). Used both on the explicit d x d problem (the plain definition of C-LOT) and
    on the small m x m problem of eq. small_problem_CLOT."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    C = np.asarray(C, dtype=np.float64)
    p, q = C.shape
    rows = scipy.sparse.kron(scipy.sparse.eye(p), np.ones((1, q)))       # (T 1)_i
    cols = scipy.sparse.kron(np.ones((1, p)), scipy.sparse.eye(q))       # (T^T 1)_j
    A_eq = scipy.sparse.vstack([rows, cols]).tocsr()
    b_eq = np.concatenate([a, b])
    res = scipy.optimize.linprog(C.ravel(), A_eq=A_eq, b_eq=b_eq, bounds=(0, None), method="highs",
                                 options={"primal_feasibility_tolerance": 1e-10,
                                          "dual_feasibility_tolerance": 1e-10})
    if res.status != 0:
        raise RuntimeError(f"LP failed: {res.message}")
    T = np.maximum(res.x.reshape(p, q), 0.0)
    return float(C.ravel() @ res.x), T


def clot(alpha: np.ndarray, beta: np.ndarray, C_blocks: np.ndarray):
    """Algorithm 1: line 1 G by eq. definition_G; line 2 the small LOT;
    lines 3-5 lift by eq. optimal_solution_problem_CLOT; line 6 expand by Lemma 1.
    Returns dict with G, A, S, T_blocks, the small value <G,S>, and the full-scale value
    n <G,S> (the reduced objective is 1/n of the full one; Theorem 1 value equality)."""
    C_blocks = np.asarray(C_blocks, dtype=np.float64)
    n = C_blocks.shape[0]
    G, A = aggregate(C_blocks)
    small, S = lot(alpha, beta, G)
    T_blocks = lift(S, A, n)
    return {"G": G, "A": A, "S": S, "T_blocks": T_blocks, "small_value": small,
            "value": n * small}


def naive_tile_lot(alpha: np.ndarray, beta: np.ndarray, C_blocks: np.ndarray) -> float:
    """The 'intuitive' strategy the paper refutes (App. A): solve OT on one
    symmetric component only (cost C_0, marginals alpha, beta) and concatenate n copies; the full
    plan is block-diagonal, so its full-scale cost is n * <C_0, S_0>."""
    C_blocks = np.asarray(C_blocks, dtype=np.float64)
    n = C_blocks.shape[0]
    v, _ = lot(alpha, beta, C_blocks[0])
    return n * v


def lot_full(alpha, beta, C_blocks):
    """Plain-definition C-LOT: LP on the explicit d x d problem (Assumption 1 inputs expanded)."""
    n = np.asarray(C_blocks).shape[0]
    return lot(expand_vector(alpha, n), expand_vector(beta, n), expand_cost(C_blocks))

