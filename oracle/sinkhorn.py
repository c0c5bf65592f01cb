"""TEST INFRASTRUCTURE (oracle) — entropic OT: full Sinkhorn on the explicit d x d problem, cyclic
Sinkhorn (Algorithm 2) in two independent forms, plan reconstruction, the Fenchel dual and the report.
Plain fp64 NumPy, log domain. See oracle/__init__.py for the import rules.

Potentials are in the paper's units: w_i = lambda log p_i, z_j = lambda log q_j. Here lambda
is written eps (BASELINE.json's letter)."""
from __future__ import annotations

import numpy as np

__all__ = ["lse", "sinkhorn_full", "cyclic_sinkhorn", "plan_blocks", "plan_full", "dual_objective",
           "report", "softmin_cost", "col_residual_after_p", "CHUNK_ELEMS"]

CHUNK_ELEMS = 1 << 23   # rows/columns are processed in chunks of independent outputs to bound memory


def lse(x: np.ndarray, axis) -> np.ndarray:
    """log sum exp over `axis`, shifted by the maximum (the definition, computed stably)."""
    mx = np.max(x, axis=axis, keepdims=True)
    mx = np.where(np.isfinite(mx), mx, 0.0)
    out = np.log(np.sum(np.exp(x - mx), axis=axis, keepdims=True)) + mx
    return np.squeeze(out, axis=axis)


# ----------------------------------------------------------------------------------------------
# full Sinkhorn on the explicit d x d problem (the plain definition of the EROT iteration)
# ----------------------------------------------------------------------------------------------
def sinkhorn_full(a, b, C, eps, iters, tol=0.0, check_every=1, record=False, g0=None):
    """Original Sinkhorn (Alg. 3 stage 2; Cuturi 2013) in the log domain of
    eq. optimal_f_sinkhorn_logdomain with n = 1:
        f_I = eps (log a_I - log sum_J exp((g_J - C_IJ)/eps))      [p <- a / (K q)]
        g_J = eps (log b_J - log sum_I exp((f_I - C_IJ)/eps))      [q <- b / (K^T p)]
    starting from q = 1 (g = 0), or from q = exp(g0/eps) (Alg. 3 line 11: stage 2 starts from the
    concatenated stage-1 scalings). Stops after `iters` iterations, or earlier when tol > 0 and the
    column residual sum_J |T^T 1 - b|_J of the row-exact plan (after the f-update) is <= tol,
    checked every `check_every` iterations. Returns (f, g, iterations_done, history)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    C = np.asarray(C, dtype=np.float64)
    g = np.zeros(C.shape[1]) if g0 is None else np.asarray(g0, dtype=np.float64).copy()
    f = np.zeros(C.shape[0])
    hist = []
    t = 0
    for t in range(1, iters + 1):
        f = eps * (np.log(a) - lse((g[None, :] - C) / eps, axis=1))
        if record or tol > 0:
            T = np.exp((f[:, None] + g[None, :] - C) / eps)
            res = float(np.abs(T.sum(0) - b).sum())
        g = eps * (np.log(b) - lse((f[:, None] - C) / eps, axis=0))
        if record:
            hist.append((f.copy(), g.copy(), res))
        if tol > 0 and t % check_every == 0 and res <= tol:
            break
    return f, g, t, hist


# ----------------------------------------------------------------------------------------------
# cyclic Sinkhorn (Algorithm 2) on the reduced problem: 2m potentials
# ----------------------------------------------------------------------------------------------
def _w_update_stream(alpha, z, C, eps):
    """eq. optimal_f_sinkhorn_logdomain with K_ij = sum_k exp(-C_ijk/eps)
    kept inside the log-sum-exp: w_i = eps (log alpha_i - log sum_{j,k} exp((z_j - C_ijk)/eps))."""
    n, m, _ = C.shape
    w = np.empty(m)
    step = max(1, CHUNK_ELEMS // (n * m))
    for i0 in range(0, m, step):
        X = (z[None, None, :] - np.asarray(C[:, i0:i0 + step, :], dtype=np.float64)) / eps
        w[i0:i0 + step] = eps * (np.log(alpha[i0:i0 + step]) - lse(X, axis=(0, 2)))
    return w


def _z_update_stream(beta, w, C, eps):
    """q-update (Alg. 2 line 5) in log form: z_j = eps (log beta_j - log sum_{i,k}
    exp((w_i - C_ijk)/eps))."""
    n, m, _ = C.shape
    z = np.empty(m)
    step = max(1, CHUNK_ELEMS // (n * m))
    for j0 in range(0, m, step):
        X = (w[None, :, None] - np.asarray(C[:, :, j0:j0 + step], dtype=np.float64)) / eps
        z[j0:j0 + step] = eps * (np.log(beta[j0:j0 + step]) - lse(X, axis=(0, 1)))
    return z


def col_residual_after_p(w, z, beta, C, eps) -> float:
    """Full-scale L1 column residual n * sum_j |c_j - beta_j| of the plan T_ijk = exp((w+z-C)/eps)
    (SURVEY Q1): c_j = sum_{i,k} T_ijk."""
    n, m, _ = C.shape
    c = np.empty(m)
    step = max(1, CHUNK_ELEMS // (n * m))
    for j0 in range(0, m, step):
        X = (w[None, :, None] + z[None, None, j0:j0 + step] - np.asarray(C[:, :, j0:j0 + step], np.float64)) / eps
        c[j0:j0 + step] = np.exp(X).sum(axis=(0, 1))
    return float(n * np.abs(c - beta).sum())


def cyclic_sinkhorn(alpha, beta, C, eps, iters, tol=0.0, check_every=1, form="stream", z0=None,
                    record=False):
    """Algorithm 2, Fast Cyclic Sinkhorn, lines 2-6, in the log domain:
        line 2: q <- 1_m                    (z = 0; or a warm start z0)
        line 4: p <- alpha / (K q)          (w-update, eq. P:403-411)
        line 5: q <- beta / (K^T p)         (z-update)
    form = "stream": the k-sum stays inside each log-sum-exp (the GPU's streaming order of work);
    form = "kernel": Alg. 2 line 1 as written, log K_ij = log sum_k exp(-C_ijk/eps) precomputed once,
                     then m x m log-sum-exps (the paper's own CPU algorithm).
    Iteration count / stopping rule as in sinkhorn_full (residual of the row-exact plan
    after the p-update, checked every `check_every` iterations; the returned state always ends with a
    q-update). Returns (w, z, iterations_done, history[(w, z, residual)])."""
    alpha = np.asarray(alpha, dtype=np.float64)
    beta = np.asarray(beta, dtype=np.float64)
    n, m, _ = C.shape
    z = np.zeros(m) if z0 is None else np.asarray(z0, dtype=np.float64).copy()
    w = np.zeros(m)
    if form == "kernel":
        logK = lse(-np.asarray(C, dtype=np.float64) / eps, axis=0)          # line 1, eq. def_Kij
    hist = []
    t = 0
    for t in range(1, iters + 1):
        if form == "stream":
            w = _w_update_stream(alpha, z, C, eps)
        else:
            w = eps * (np.log(alpha) - lse(logK + z[None, :] / eps, axis=1))
        res = None
        if record or tol > 0:
            if form == "stream":
                res = col_residual_after_p(w, z, beta, C, eps)
            else:   # same quantity through K: c_j = sum_i K_ij p_i q_j
                c = np.exp(logK + (w[:, None] + z[None, :]) / eps).sum(0)
                res = float(n * np.abs(c - beta).sum())
        if form == "stream":
            z = _z_update_stream(beta, w, C, eps)
        else:
            z = eps * (np.log(beta) - lse(logK + w[:, None] / eps, axis=0))
        if record:
            hist.append((w.copy(), z.copy(), res))
        if tol > 0 and t % check_every == 0 and res <= tol:
            break
    return w, z, t, hist


# ----------------------------------------------------------------------------------------------
# plan, dual, report
# ----------------------------------------------------------------------------------------------
def plan_blocks(w, z, C, eps) -> np.ndarray:
    """Alg. 2 lines 7-9: T_ijk = p_i q_j exp(-C_ijk/eps) = exp((w_i + z_j - C_ijk)/eps),
    the optimality condition eq. optimality_condition with (phi*)'(y) = exp(y/eps)."""
    C = np.asarray(C, dtype=np.float64)
    return np.exp((w[None, :, None] + z[None, None, :] - C) / eps)


def plan_full(f, g, C, eps) -> np.ndarray:
    """T = diag(p) K diag(q) (Alg. 3 line 14) for the explicit problem."""
    return np.exp((f[:, None] + g[None, :] - np.asarray(C, dtype=np.float64)) / eps)


def dual_objective(w, z, alpha, beta, C, eps) -> float:
    """Reduced Fenchel dual, eq. dual_problem_cyclic_ROT with phi*(y) = lambda exp(y/lambda)
    (P:393): <w, alpha> + <z, beta> - sum_{k,i,j} eps exp((w_i + z_j - C_ijk)/eps)."""
    T = plan_blocks(w, z, C, eps)
    return float(w @ alpha + z @ beta - eps * T.sum())


def softmin_cost(C, eps) -> np.ndarray:
    """G^eps_ij = -eps log sum_k exp(-C_ijk/eps) = -eps log K_ij (eq. def_Kij)."""
    return -eps * lse(-np.asarray(C, dtype=np.float64) / eps, axis=0)


def report(w, z, alpha, beta, C, eps) -> dict:
    """Full-scale quantities of the plan reconstructed from (w, z) (all x n: the reduced objective is
    1/n of the full one):
      objective  = transport cost n * sum_k <C_k, T_k>        (Table 1's 'Obj. value')
      reg_primal = objective + n * eps * sum T (log T - 1)      (eq. problem_CROT with eq. reg_for_entropy_ROT)
      dual       = n * (<w,alpha> + <z,beta> - eps sum T)       (eq. dual_problem_cyclic_ROT, Q4)
      row_l1     = sum_I |T 1_d - a|_I   = n * sum_i |r_i - alpha_i|
      col_l1     = sum_J |T^T 1_d - b|_J = n * sum_j |c_j - beta_j|
      col_l2     = ||T^T 1_d - b||_2     (the marginal error of Sec. 6.1)
      mass       = sum of the full plan = n * sum T_ijk
    plus the reduced row/column sums r (= sum_{j,k} T_ijk) and c (= sum_{i,k} T_ijk)."""
    C64 = np.asarray(C, dtype=np.float64)
    n = C64.shape[0]
    T = plan_blocks(w, z, C64, eps)
    logT = (w[None, :, None] + z[None, None, :] - C64) / eps
    r = T.sum(axis=(0, 2))
    c = T.sum(axis=(0, 1))
    transport = float((C64 * T).sum())
    ent = float((T * (logT - 1.0)).sum())
    return {
        "objective": n * transport,
        "reg_primal": n * (transport + eps * ent),
        "dual": n * float(w @ alpha + z @ beta - eps * T.sum()),
        "row_l1": float(n * np.abs(r - alpha).sum()),
        "col_l1": float(n * np.abs(c - beta).sum()),
        "col_l2": float(np.sqrt(n * ((c - beta) ** 2).sum())),
        "mass": float(n * T.sum()),
        "r": r, "c": c,
    }
