"""TEST INFRASTRUCTURE (oracle) — structure of the cyclic problem: expansion, symmetrisation,
aggregation G / argmin, lift. Plain fp64 NumPy. See oracle/__init__.py for the import rules."""
from __future__ import annotations

import numpy as np

__all__ = ["expand_vector", "expand_cost", "expand_plan", "expand_plan_rows", "block_shift_permutation", "symmetrize",
           "aggregate", "lift", "fold_average", "is_block_circulant"]


def expand_vector(v: np.ndarray, n: int) -> np.ndarray:
    """a = (alpha; alpha; ...; alpha), n copies (Assumption 1, eq. assumption_for_input_vectors,
    P:143-158)."""
    return np.concatenate([np.asarray(v, dtype=np.float64)] * n)


def expand_cost(C_blocks: np.ndarray) -> np.ndarray:
    """Block-circulant d x d matrix of eq. blkstr_cost: the first block row is
    (C_0, C_1, ..., C_{n-1}) and each following block row is the previous one shifted right by one
    block, i.e. block (r, s) = C_{(s - r) mod n}. Written as explicit loops over blocks."""
    C_blocks = np.asarray(C_blocks, dtype=np.float64)
    n, m, _ = C_blocks.shape
    d = n * m
    out = np.empty((d, d), dtype=np.float64)
    for r in range(n):
        for s in range(n):
            out[r * m:(r + 1) * m, s * m:(s + 1) * m] = C_blocks[(s - r) % n]
    return out


def expand_plan(T_blocks: np.ndarray) -> np.ndarray:
    """The d x d plan of Lemma 1, eq. blkstr_optimal_solution: same circulant placement as
    the cost (Alg. 1 line 6 'Compute T by Lemma 1'; Alg. 2 line 10). Keeps the input
    dtype (pure placement, no arithmetic)."""
    T_blocks = np.asarray(T_blocks)
    n, m, _ = T_blocks.shape
    d = n * m
    out = np.empty((d, d), dtype=T_blocks.dtype)
    for r in range(n):
        for s in range(n):
            out[r * m:(r + 1) * m, s * m:(s + 1) * m] = T_blocks[(s - r) % n]
    return out


def expand_plan_rows(T_blocks: np.ndarray, rows) -> np.ndarray:
    """Selected rows I of the d x d plan of Lemma 1 without building the whole plan: row
    I = r*m + i is (T_{(0 - r) mod n}[i], T_{(1 - r) mod n}[i], ..., T_{(n-1 - r) mod n}[i]), the same
    placement block (r, s) = T_{(s - r) mod n} as expand_plan, written out per row. For sampling plans
    too large for the host (C4: d = 65536)."""
    T_blocks = np.asarray(T_blocks)
    n, m, _ = T_blocks.shape
    out = np.empty((len(rows), n * m), dtype=T_blocks.dtype)
    for q, I in enumerate(rows):
        r, i = divmod(int(I), m)
        for s in range(n):
            out[q, s * m:(s + 1) * m] = T_blocks[(s - r) % n][i]
    return out


def block_shift_permutation(n: int, m: int) -> np.ndarray:
    """P of eq. A2: identity blocks on the block sub-diagonal and in the top-right corner."""
    d = n * m
    P = np.zeros((d, d))
    I = np.eye(m)
    for r in range(n):
        s = (r - 1) % n
        P[r * m:(r + 1) * m, s * m:(s + 1) * m] = I
    return P


def symmetrize(T: np.ndarray, n: int) -> np.ndarray:
    """T* = (1/n) sum_k P^k T' (P^k)^T, eq. A1, with P materialised (proof device)."""
    T = np.asarray(T, dtype=np.float64)
    d = T.shape[0]
    m = d // n
    P = block_shift_permutation(n, m)
    acc = np.zeros_like(T)
    Pk = np.eye(d)
    for _ in range(n):
        acc += Pk @ T @ Pk.T
        Pk = P @ Pk
    return acc / n


def is_block_circulant(M: np.ndarray, n: int) -> bool:
    """P M P^T == M exactly, the fixed-point property shown at the end of Lemma 1's proof."""
    m = M.shape[0] // n
    P = block_shift_permutation(n, m)
    return bool(np.array_equal(P @ M @ P.T, M))


def aggregate(C_blocks: np.ndarray):
    """G_ij = min_k C_ijk (eq. definition_G) and the SMALLEST minimising k
    (eq. optimal_solution_problem_CLOT: k = min(argmin_k C_ijk); tie remark P:291).
    G is taken as C[A_ij][i][j], so the sign of a zero is the one stored at the chosen k
    (SURVEY Q8). Works for [n][m][m] or [B][n][m][m]; keeps the input dtype (comparisons only)."""
    C = np.asarray(C_blocks)
    kaxis = C.ndim - 3
    A = np.argmin(C, axis=kaxis)                                 # numpy: first occurrence of the min
    G = np.take_along_axis(C, np.expand_dims(A, kaxis), axis=kaxis).squeeze(kaxis)
    if np.isnan(C).any():
        raise ValueError("non-finite cost (NaN)")
    return G, A.astype(np.int32)


def lift(S: np.ndarray, A: np.ndarray, n: int) -> np.ndarray:
    """T*_ijk = S*_ij if k = A_ij else 0 (eq. optimal_solution_problem_CLOT). Keeps S's dtype."""
    S = np.asarray(S)
    m = S.shape[0]
    T = np.zeros((n, m, m), dtype=S.dtype)
    for k in range(n):
        T[k][A == k] = S[A == k]
    return T


def fold_average(v: np.ndarray, n: int) -> np.ndarray:
    """alpha_i = (1/n) sum_k a_{i + m k} (Alg. 3 lines 2-3)."""
    v = np.asarray(v, dtype=np.float64)
    m = v.shape[0] // n
    return v.reshape(n, m).sum(0) / n
