"""TEST INFRASTRUCTURE (oracle) — NEXT-2: the two-stage Sinkhorn algorithm for C-EROT with approximate
cyclic symmetry (Algorithm 3; App. F stopping rules P:792-795). Plain fp64 NumPy built from the
oracle's own steps. See oracle/__init__.py for the import rules."""
from __future__ import annotations

import numpy as np

from .core import expand_cost, expand_vector, fold_average
from .sinkhorn import cyclic_sinkhorn, sinkhorn_full

__all__ = ["two_stage_sinkhorn"]


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
