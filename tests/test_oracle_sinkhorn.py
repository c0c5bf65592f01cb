"""Pins for the oracle's EROT side: full Sinkhorn, cyclic Sinkhorn (both forms), plan, dual, report.

Pins: closed forms (C = 0, m = 1, the 2 x 2 fixed point of S:372, eps -> infinity, the dual at the
origin), the iterate identity full (explicit d x d) == tiled reduced at every iteration (P:161-168 with
P:398-400), the textbook reduction to m x m EROT with the soft-min cost, strong duality and monotone
dual ascent, row exactness after the p-update, divisor invariance, the
objective factor n, and the Table 1 paired excess."""
import math

import numpy as np
import pytest

import oracle
import synthetic
from conftest import golden


def _full(p):
    n = p.n
    return (oracle.expand_vector(p.alpha, n), oracle.expand_vector(p.beta, n),
            oracle.expand_cost(p.C))


# ------------------------------------------------------------------------------------ closed forms
def test_closed_form_zero_cost():
    """C = 0: one iteration gives T_k = alpha beta^T for every k (rank-one balancing)."""
    rng = np.random.default_rng(0)
    n, m = 3, 5
    alpha = rng.dirichlet(np.ones(m)) / n
    beta = rng.dirichlet(np.ones(m)) / n
    C = np.zeros((n, m, m))
    w, z, _, _ = oracle.cyclic_sinkhorn(alpha, beta, C, 0.3, 1)
    T = oracle.plan_blocks(w, z, C, 0.3)
    for k in range(n):
        assert np.allclose(T[k], np.outer(alpha, beta), rtol=1e-13, atol=0)


def test_closed_form_m1():
    """m = 1: after one iteration T_k = alpha exp(-C_k/eps) / sum_k' exp(-C_k'/eps)."""
    C = np.array([[[0.0]], [[1.0]], [[0.25]]])
    eps = 0.7
    alpha = beta = np.array([1 / 3])
    w, z, _, _ = oracle.cyclic_sinkhorn(alpha, beta, C, eps, 1)
    T = oracle.plan_blocks(w, z, C, eps)[:, 0, 0]
    e = np.exp(-C[:, 0, 0] / eps)
    assert np.allclose(T, alpha[0] * e / e.sum(), rtol=1e-14)


def test_closed_form_2x2_fixed_point():
    """d = 2, a = b = (0.5, 0.5), C = [[0, c], [c, 0]] -> diagonal mass 0.5 / (1 + e^{-c/l}).
    As a cyclic problem: n = 2, m = 1, blocks [0], [c]; T_0 is the diagonal entry."""
    c, lam = 1.3, 0.5
    diag = 0.5 / (1 + math.exp(-c / lam))
    f, g, _, _ = oracle.sinkhorn_full([0.5, 0.5], [0.5, 0.5], [[0, c], [c, 0]], lam, 50)
    T = oracle.plan_full(f, g, [[0, c], [c, 0]], lam)
    assert abs(T[0, 0] - diag) <= 1e-15 and abs(T[1, 1] - diag) <= 1e-15
    w, z, _, _ = oracle.cyclic_sinkhorn([0.5], [0.5], np.array([[[0.0]], [[c]]]), lam, 50)
    Tb = oracle.plan_blocks(w, z, np.array([[[0.0]], [[c]]]), lam)
    assert abs(Tb[0, 0, 0] - diag) <= 1e-15


def test_kernel_limits_and_dual_at_origin():
    rng = np.random.default_rng(5)
    C = rng.random((4, 3, 3))
    # eps -> infinity: K -> n, i.e. the soft-min cost G^eps -> -eps log n
    big = 1e8
    assert np.allclose(oracle.softmin_cost(C, big) / big, -math.log(4), atol=1e-7)
    # w = z = 0: dual = -eps sum exp(-C/eps); m = n = 1, C = 0, eps = 1 -> -1
    alpha = beta = np.full(3, 1 / 12)
    d0 = oracle.dual_objective(np.zeros(3), np.zeros(3), alpha, beta, C, 0.4)
    assert math.isclose(d0, -0.4 * np.exp(-C / 0.4).sum(), rel_tol=1e-15)
    assert oracle.dual_objective(np.zeros(1), np.zeros(1), np.ones(1), np.ones(1), np.zeros((1, 1, 1)), 1.0) == -1.0


def test_softmin_sandwich():
    """G - eps log n <= G^eps <= G (links eq. definition_G to eq. def_Kij)."""
    p = synthetic.c2_ring()
    G, _ = oracle.aggregate(p.C.astype(np.float64))
    for eps in (1e-3, 1e-2, 1e-1, 1.0):
        Ge = oracle.softmin_cost(p.C, eps)
        assert np.all(Ge <= G + 1e-12) and np.all(Ge >= G - eps * math.log(p.n) - 1e-12)


# ---------------------------------------------------------------- reduced == full, two forms
def test_iterate_identity_full_vs_reduced_c1():
    """Periodic q: sum_s K_{(s-r) mod n} q_hat = K_hat q_hat, so full Sinkhorn on the explicit problem
    from q = 1_d equals the tiled reduced iterates at EVERY iteration (SURVEY [V1])."""
    p = synthetic.c1_tiny()
    a, b, C = _full(p)
    eps = float(p.eps[0])
    f, g, _, hf = oracle.sinkhorn_full(a, b, C, eps, 60, record=True)
    w, z, _, hc = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, eps, 60, record=True)
    for (ff, gg, rf), (ww, zz, rc) in zip(hf, hc):
        assert np.abs(ff - np.tile(ww, p.n)).max() <= 1e-14
        assert np.abs(gg - np.tile(zz, p.n)).max() <= 1e-14
        assert abs(rf - rc) <= 1e-14


def test_stream_equals_kernel_form():
    """Alg. 2 as written (K precomputed) vs the streaming k-sum: same iterates."""
    p = synthetic.c2_ring(eps_factor=1e-2)
    eps = float(p.eps[0])
    w1, z1, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, eps, 40, form="stream")
    w2, z2, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, eps, 40, form="kernel")
    assert np.abs(w1 - w2).max() <= 1e-12 * max(1, np.abs(w1).max())
    assert np.abs(z1 - z2).max() <= 1e-12 * max(1, np.abs(z1).max())


def test_textbook_softmin_reduction():
    """Reduced C-EROT == plain m x m EROT on (alpha, beta, G^eps), G^eps = -eps log sum_k e^{-C_k/eps};
    the lift is T_ijk = S_ij softmax_k(-C_ijk/eps) (SURVEY §8(c) textbook special case)."""
    p = synthetic.random_cyclic(seed=3, n=5, m=7, eps=0.2)
    eps = 0.2
    w, z, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, eps, 200)
    Ge = oracle.softmin_cost(p.C, eps)
    f, g, _, _ = oracle.sinkhorn_full(p.alpha, p.beta, Ge, eps, 200)
    assert np.abs(w - f).max() <= 1e-13 and np.abs(z - g).max() <= 1e-13
    S = oracle.plan_full(f, g, Ge, eps)
    soft = np.exp(-p.C / eps) / np.exp(-p.C / eps).sum(0, keepdims=True)
    assert np.allclose(S[None] * soft, oracle.plan_blocks(w, z, p.C, eps), rtol=1e-12, atol=1e-300)


# ---------------------------------------------------------------- invariants
def test_duality_monotone_ascent_and_row_exactness():
    p = synthetic.random_cyclic(seed=9, n=6, m=10, eps=0.05)
    eps = 0.05
    w, z, t, hist = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, eps, 3000, tol=1e-14, record=True)
    assert t < 3000
    duals = []
    zprev = np.zeros(p.m)
    for (ww, zz, _) in hist:
        duals.append(oracle.dual_objective(ww, zprev, p.alpha, p.beta, p.C, eps))   # after p-update
        T = oracle.plan_blocks(ww, zprev, p.C, eps)
        assert np.abs(T.sum(axis=(0, 2)) - p.alpha).max() <= 1e-15                 # row-exact
        duals.append(oracle.dual_objective(ww, zz, p.alpha, p.beta, p.C, eps))      # after q-update
        zprev = zz
    assert all(b >= a - 1e-15 for a, b in zip(duals, duals[1:]))                    # alternating max
    rep = oracle.report(w, z, p.alpha, p.beta, p.C, eps)
    assert abs(rep["reg_primal"] - rep["dual"]) <= 1e-13                            # strong duality
    assert rep["col_l1"] <= 1e-13 and rep["row_l1"] <= 1e-12


def test_objective_factor_n_and_gauge():
    """the objective of the reduced problem is 1/n of the full one; the gauge (w + c, z - c)
    leaves the plan and the dual unchanged."""
    p = synthetic.c1_tiny()
    eps = float(p.eps[0])
    w, z, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, eps, 2)  # not yet converged
    rep = oracle.report(w, z, p.alpha, p.beta, p.C, eps)
    Tfull = oracle.expand_plan(oracle.plan_blocks(w, z, p.C, eps))
    a, b, Cfull = _full(p)
    assert math.isclose((Cfull * Tfull).sum(), rep["objective"], rel_tol=1e-13)
    # after a q-update the columns are exact up to rounding, the rows carry the residual
    assert rep["row_l1"] > 1e-6
    assert math.isclose(np.abs(Tfull.sum(1) - a).sum(), rep["row_l1"], rel_tol=1e-9)
    assert abs(np.abs(Tfull.sum(0) - b).sum() - rep["col_l1"]) <= 1e-15
    assert abs(np.sqrt(((Tfull.sum(0) - b) ** 2).sum()) - rep["col_l2"]) <= 1e-15
    rep2 = oracle.report(w + 0.37, z - 0.37, p.alpha, p.beta, p.C, eps)
    assert math.isclose(rep2["objective"], rep["objective"], rel_tol=1e-12)
    assert math.isclose(rep2["dual"], rep["dual"], rel_tol=1e-12)


def test_c1_converges_and_matches_full():
    """C1 to n*sum|c - beta| <= 1e-9 checked every iteration; the converged plan's transport cost equals
    full Sinkhorn's on the explicit problem, and exceeds the C-LOT value (P:515 vs P:539 ordering)."""
    p = synthetic.c1_tiny()
    eps = float(p.eps[0])
    w, z, t, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, eps, 100000, tol=1e-9)
    a, b, C = _full(p)
    f, g, tf, _ = oracle.sinkhorn_full(a, b, C, eps, 100000, tol=1e-9)
    assert t == tf
    rep = oracle.report(w, z, p.alpha, p.beta, p.C, eps)
    Tf = oracle.plan_full(f, g, C, eps)
    assert math.isclose(rep["objective"], (C * Tf).sum(), rel_tol=1e-12)
    assert rep["col_l1"] <= 1e-9
    assert rep["objective"] > oracle.clot(p.alpha, p.beta, p.C)["value"]


def test_eps_trend_toward_clot():
    """eps -> 0: the EROT transport cost decreases toward the C-LOT value (SURVEY [V11])."""
    p = synthetic.random_cyclic(seed=21, n=4, m=12)
    lotv = oracle.clot(p.alpha, p.beta, p.C)["value"]
    costs = []
    for eps in (0.3, 0.1, 0.03, 0.01):
        w, z, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, eps, 20000, tol=1e-12, form="kernel")
        costs.append(oracle.report(w, z, p.alpha, p.beta, p.C, eps)["objective"])
    assert all(c2 < c1 for c1, c2 in zip(costs, costs[1:]))
    assert all(c > lotv for c in costs) and costs[-1] - lotv < 0.1 * (costs[0] - lotv)


def test_divisor_invariance_erot():
    """every divisor n of n_max gives the same EROT objective (same explicit problem)."""
    p = synthetic.appd_synthetic(seed=1, d=24, n_max=6)
    a = oracle.expand_vector(p.alpha, 6)
    b = oracle.expand_vector(p.beta, 6)
    Cfull = oracle.expand_cost(p.C)
    vals = []
    for n in (1, 2, 3, 6):
        m = 24 // n
        blocks = np.stack([Cfull[0:m, s * m:(s + 1) * m] for s in range(n)])
        w, z, _, _ = oracle.cyclic_sinkhorn(a[:m], b[:m], blocks, 0.5, 5000, tol=1e-13)
        vals.append(oracle.report(w, z, a[:m], b[:m], blocks, 0.5)["objective"])
    assert max(vals) - min(vals) <= 1e-11


@pytest.mark.slow
def test_table1_paired_excess_d5000():
    """Table 1: mean over 20 App. D instances (d = 5000, n = 50, lambda = 0.5) of
    'cyclic Sinkhorn transport cost - cyclic network simplex value' = 0.199 in the paper; the per-instance
    values are not reproducible, so the check is |mean - 0.199| <= 0.02."""
    g = golden("table1_excess.json")["d5000"]
    ex = []
    for seed in range(20):
        p = synthetic.appd_synthetic(seed=seed, d=5000, n_max=50)
        lotv = oracle.clot(p.alpha, p.beta, p.C)["value"]
        w, z, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, 0.5, 20000, tol=1e-10, check_every=10,
                                            form="kernel")
        ex.append(oracle.report(w, z, p.alpha, p.beta, p.C, 0.5)["objective"] - lotv)
    assert all(e > 0 for e in ex)
    assert abs(np.mean(ex) - g["paper_excess"]) <= g["threshold"], np.mean(ex)


@pytest.mark.slow
def test_table1_paired_excess_d10000():
    """As above at d = 10000 (m = 200): paper 6.745 - 6.526 = 0.219."""
    g = golden("table1_excess.json")["d10000"]
    ex = []
    for seed in range(20):
        p = synthetic.appd_synthetic(seed=seed, d=10000, n_max=50)
        lotv = oracle.clot(p.alpha, p.beta, p.C)["value"]
        w, z, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, 0.5, 20000, tol=1e-10, check_every=10,
                                            form="kernel")
        ex.append(oracle.report(w, z, p.alpha, p.beta, p.C, 0.5)["objective"] - lotv)
    assert abs(np.mean(ex) - g["paper_excess"]) <= g["threshold"], np.mean(ex)
