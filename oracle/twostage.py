"""TEST INFRASTRUCTURE (oracle) — NEXT-2: the two-stage Sinkhorn algorithm for C-EROT with approximate
cyclic symmetry (Algorithm 3; App. F stopping rules P:792-795). Plain fp64 NumPy built from the
oracle's own steps. See oracle/__init__.py for the import rules."""
from __future__ import annotations

import numpy as np

from .core import expand_cost, expand_vector, fold_average
from .sinkhorn import cyclic_sinkhorn, lse, sinkhorn_full

__all__ = ["two_stage_sinkhorn", "two_stage_sinkhorn_gap", "entropic_objective_full"]


def two_stage_sinkhorn(a, b, C_blocks, eps, iters1, iters2, tol1=0.0, tol2=0.0, check_every=1):
    """Algorithm 3, inputs a, b in Delta^d (approximately periodic), C block-circulant with the
    n blocks C_blocks (Assumption 1 holds for C strictly):
      lines 2-5   alpha_i = (1/n) sum_k a_{i+mk}, beta_i likewise (the fold averages);
      lines 6-10  cyclic Sinkhorn (Alg. 2) on (alpha, beta, C_blocks) from q^ = 1 for `iters1` iterations or
                  until its monitor <= tol1 (SURVEY Q19 reading: the same monitor as Alg. 2, not App. F's l2);
      line 11     p, q = the n concatenated p^, q^ (f = tile(w), g = tile(z) in the log domain);
      lines 12-16 the original Sinkhorn on the explicit d x d problem (a, b, C) from that start, `iters2`
                  iterations or until its column residual <= tol2.
    Returns (f, g, stage-1 iterations, stage-2 iterations) with f, g the d-length potentials (lambda log p)."""
    C_blocks = np.asarray(C_blocks, dtype=np.float64)
    n = C_blocks.shape[0]
    alpha = fold_average(a, n)
    beta = fold_average(b, n)
    w, z, t1, _ = cyclic_sinkhorn(alpha, beta, C_blocks, eps, iters1, tol=tol1, check_every=check_every,
                                  form="kernel")
    f, g, t2, _ = sinkhorn_full(a, b, expand_cost(C_blocks), eps, iters2, tol=tol2, check_every=check_every,
                                g0=expand_vector(z, n))
    return f, g, t1, t2


def entropic_objective_full(T, C, eps) -> float:
    """The C-EROT objective of an explicit plan (eq. problem_CROT with the entropic regulariser, eq.
    reg_for_entropy_ROT, in the form the oracle's report uses): <C, T> + eps sum_IJ T_IJ (log T_IJ - 1),
    with 0 log 0 = 0."""
    T = np.asarray(T, dtype=np.float64)
    pos = T > 0
    return float((np.asarray(C, dtype=np.float64) * T).sum() + eps * (T[pos] * (np.log(T[pos]) - 1.0)).sum())


def two_stage_sinkhorn_gap(a, b, C_blocks, eps, iters1, iters2, obj_ref, tol_obj, tol1=0.0, check_every=1):
    """Algorithm 3 with App. F's stage-2 stopping rule: "we then run the original Sinkhorn algorithm
    until the difference between its objective function value and the value obtained by directly solving
    [the problem] using the original Sinkhorn algorithm is below 1.0e-4". Stage 1 as two_stage_sinkhorn;
    stage 2: one original Sinkhorn iteration at a time (p-update, q-update), and after every
    `check_every`-th iteration the objective (entropic_objective_full, DESIGN reading Q19: the regularised
    primal) of T = diag(p) K diag(q); stop when |objective - obj_ref| < tol_obj or after iters2 iterations.
    Returns (f, g, stage-1 iterations, stage-2 iterations, last measured gap or None)."""
    C_blocks = np.asarray(C_blocks, dtype=np.float64)
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    n = C_blocks.shape[0]
    w, z, t1, _ = cyclic_sinkhorn(fold_average(a, n), fold_average(b, n), C_blocks, eps, iters1, tol=tol1,
                                  check_every=check_every, form="kernel")
    C = expand_cost(C_blocks)
    g = expand_vector(z, n)
    f = np.zeros_like(g)
    gap = None
    t2 = 0
    for t2 in range(1, iters2 + 1):
        f = eps * (np.log(a) - lse((g[None, :] - C) / eps, axis=1))
        g = eps * (np.log(b) - lse((f[:, None] - C) / eps, axis=0))
        if t2 % check_every == 0:
            T = np.exp((f[:, None] + g[None, :] - C) / eps)
            gap = abs(entropic_objective_full(T, C, eps) - obj_ref)
            if gap < tol_obj:
                break
    return f, g, t1, t2, gap
