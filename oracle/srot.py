"""TEST INFRASTRUCTURE (oracle) — C-SROT: strongly convex regularised OT with cyclic symmetry through its
2m-variable Fenchel dual (Theorem 2) and alternating maximisation with per-coordinate safeguarded
Newton. Plain fp64 NumPy. See oracle/__init__.py for the import rules.

Regularisers:
  ("entropic", lam): phi(x) = lam x (log x - 1), phi*(y) = lam e^{y/lam}, (phi*)'(y) = e^{y/lam}
  ("squared", gam):  phi(x) = x^2 / (2 gam) for x >= 0, phi*(y) = gam/2 max(y,0)^2, (phi*)'(y) = gam max(y,0)
Potentials w, z are in cost units (not eps-scaled)."""
from __future__ import annotations

import numpy as np

__all__ = ["conj", "conj_prime", "phi", "srot_dual", "partial_w", "partial_z", "coordinate_solve",
           "alternating_maximize", "srot_plan", "srot_report"]


def conj(y, reg):
    kind, par = reg
    y = np.asarray(y, dtype=np.float64)
    if kind == "entropic":
        return par * np.exp(y / par)
    return 0.5 * par * np.maximum(y, 0.0) ** 2


def conj_prime(y, reg):
    kind, par = reg
    y = np.asarray(y, dtype=np.float64)
    if kind == "entropic":
        return np.exp(y / par)
    return par * np.maximum(y, 0.0)


def phi(x, reg):
    kind, par = reg
    x = np.asarray(x, dtype=np.float64)
    if kind == "entropic":
        with np.errstate(divide="ignore", invalid="ignore"):
            return np.where(x > 0, par * x * (np.log(np.where(x > 0, x, 1.0)) - 1.0), 0.0)
    return x * x / (2.0 * par)


def srot_dual(w, z, alpha, beta, C, reg) -> float:
    """eq. dual_problem_cyclic_ROT: <w,alpha> + <z,beta> - sum_{k,i,j} phi*(w_i + z_j - C_ijk)."""
    C = np.asarray(C, dtype=np.float64)
    return float(w @ alpha + z @ beta - conj(w[None, :, None] + z[None, None, :] - C, reg).sum())


def partial_w(w, z, alpha, C, reg) -> np.ndarray:
    """eq. derivative_of_objective_function for every i: alpha_i - sum_{k,j} (phi*)'(w_i+z_j-C_ijk)."""
    C = np.asarray(C, dtype=np.float64)
    return alpha - conj_prime(w[None, :, None] + z[None, None, :] - C, reg).sum(axis=(0, 2))


def partial_z(w, z, beta, C, reg) -> np.ndarray:
    C = np.asarray(C, dtype=np.float64)
    return beta - conj_prime(w[None, :, None] + z[None, None, :] - C, reg).sum(axis=(0, 1))


def coordinate_solve(target, b, reg, x0=0.0, tol=1e-14, max_iter=200):
    """Solve target = sum_l (phi*)'(x - b_l) for x (one coordinate of P:374-380; the right side is
    monotonically increasing in x): safeguarded Newton with a bisection fallback.
    b: the breakpoints C_ijk - z_j (for w_i) or C_ijk - w_i (for z_j)."""
    b = np.asarray(b, dtype=np.float64).ravel()
    f = lambda x: conj_prime(x - b, reg).sum() - target            # increasing in x
    kind, par = reg
    if kind == "entropic":   # closed form (eq. optimal_f_sinkhorn_logdomain), as the Newton limit
        mx = np.max(-b / par)
        return par * (np.log(target) - (mx + np.log(np.exp(-b / par - mx).sum())))
    lo, hi = x0 - 1.0, x0 + 1.0
    while f(lo) > 0:
        lo -= 2 * (hi - lo)
    while f(hi) < 0:
        hi += 2 * (hi - lo)
    x = hi
    for _ in range(max_iter):
        fx = f(x)
        if abs(fx) <= tol * max(1.0, target):
            break
        if fx > 0:
            hi = x
        else:
            lo = x
        d = par * np.count_nonzero(x - b > 0)                    # f'(x) (a subgradient at breakpoints)
        xn = x - fx / d if d > 0 else 0.5 * (lo + hi)
        if not (lo < xn < hi):                                  # safeguard: bisection
            xn = 0.5 * (lo + hi)
        x = xn
    return x


def alternating_maximize(alpha, beta, C, reg, sweeps, tol=0.0, check_every=1, z0=None, record=False):
    """Alternating maximisation of the dual: maximise over w with z fixed (every w_i independently,
    P:375-380), then over z with w fixed; z = 0 start. Stops after `sweeps` or when the full-scale L1 column
    residual of the row-exact plan after the w-step is <= tol (checked every check_every sweeps; same rule as
    the cyclic Sinkhorn oracle). Returns (w, z, sweeps_done, history[(w, z, residual)])."""
    C = np.asarray(C, dtype=np.float64)
    n, m, _ = C.shape
    alpha = np.asarray(alpha, np.float64)
    beta = np.asarray(beta, np.float64)
    z = np.zeros(m) if z0 is None else np.asarray(z0, np.float64).copy()
    w = np.zeros(m)
    hist = []
    t = 0
    for t in range(1, sweeps + 1):
        w = np.array([coordinate_solve(alpha[i], C[:, i, :] - z[None, :], reg) for i in range(m)])
        T = conj_prime(w[None, :, None] + z[None, None, :] - C, reg)
        res = float(n * np.abs(T.sum(axis=(0, 1)) - beta).sum())
        z = np.array([coordinate_solve(beta[j], C[:, :, j] - w[None, :], reg) for j in range(m)])
        if record:
            hist.append((w.copy(), z.copy(), res))
        if tol > 0 and t % check_every == 0 and res <= tol:
            break
    return w, z, t, hist


def srot_plan(w, z, C, reg) -> np.ndarray:
    """eq. optimality_condition: T_ijk = (phi*)'(w_i + z_j - C_ijk)."""
    return conj_prime(w[None, :, None] + z[None, None, :] - np.asarray(C, np.float64), reg)


def srot_report(w, z, alpha, beta, C, reg) -> dict:
    """Full-scale (x n) transport cost, regularised primal, dual, residuals, mass of the plan."""
    C64 = np.asarray(C, dtype=np.float64)
    n = C64.shape[0]
    T = srot_plan(w, z, C64, reg)
    r = T.sum(axis=(0, 2))
    c = T.sum(axis=(0, 1))
    transport = float((C64 * T).sum())
    return {"objective": n * transport, "reg_primal": n * (transport + float(phi(T, reg).sum())),
            "dual": n * srot_dual(w, z, alpha, beta, C64, reg), "row_l1": float(n * np.abs(r - alpha).sum()),
            "col_l1": float(n * np.abs(c - beta).sum()), "mass": float(n * T.sum()), "r": r, "c": c}
