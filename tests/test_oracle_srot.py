"""Pins for the oracle's C-SROT machinery (Theorem 2; NEXT-3).

* S:289 worked example (squared regulariser, m = n = 1: w = 1);
* the entropic coordinate solve reproduces the closed form of P:403-411, so alternating maximisation with the
  entropic regulariser reproduces the cyclic Sinkhorn oracle iterate for iterate;
* partial_w / partial_z agree with centred finite differences of the dual;
* the dual never decreases across half-sweeps (alternating maximisation);
* strong duality and feasibility at convergence;
* Lemma 1 + Theorem 2 reduction: the reduced squared-regularised problem has the same optimal value (x n) as
  the explicit d x d problem, solved independently by a generic constrained optimiser (SciPy SLSQP)."""
import math

import numpy as np
import pytest
import scipy.optimize

import oracle
import synthetic


def test_spec_example_squared():
    # squared regulariser, m = n = 1, C = [[0]], z = 0, gamma = 1, alpha = 1 -> w = 1
    w = oracle.coordinate_solve(1.0, np.array([0.0]), ("squared", 1.0))
    assert abs(w - 1.0) < 1e-14


def test_entropic_coordinate_solve_is_sinkhorn():
    p = synthetic.random_cyclic(seed=2, n=4, m=9, eps=0.3)
    w1, z1, _, _ = oracle.alternating_maximize(p.alpha, p.beta, p.C, ("entropic", 0.3), 25)
    w2, z2, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, 0.3, 25)
    assert np.abs(w1 - w2).max() < 1e-13 and np.abs(z1 - z2).max() < 1e-13


@pytest.mark.parametrize("reg", [("squared", 0.7), ("entropic", 0.4)])
def test_gradients_match_finite_differences(reg):
    rng = np.random.default_rng(3)
    p = synthetic.random_cyclic(seed=4, n=3, m=5)
    for _ in range(20):
        w, z = rng.normal(size=5) * 0.5, rng.normal(size=5) * 0.5
        g = oracle.partial_w(w, z, p.alpha, p.C, reg)
        h = 1e-5
        for i in range(5):
            e = np.zeros(5)
            e[i] = h
            fd = (oracle.srot_dual(w + e, z, p.alpha, p.beta, p.C, reg) -
                  oracle.srot_dual(w - e, z, p.alpha, p.beta, p.C, reg)) / (2 * h)
            assert abs(fd - g[i]) <= 1e-6 * max(1.0, abs(g[i]))
        gz = oracle.partial_z(w, z, p.beta, p.C, reg)
        for j in range(5):
            e = np.zeros(5)
            e[j] = h
            fd = (oracle.srot_dual(w, z + e, p.alpha, p.beta, p.C, reg) -
                  oracle.srot_dual(w, z - e, p.alpha, p.beta, p.C, reg)) / (2 * h)
            assert abs(fd - gz[j]) <= 1e-6 * max(1.0, abs(gz[j]))


def test_squared_monotone_ascent_duality_and_feasibility():
    p = synthetic.random_cyclic(seed=11, n=4, m=7)
    reg = ("squared", 0.5)
    w, z, t, hist = oracle.alternating_maximize(p.alpha, p.beta, p.C, reg, 5000, tol=1e-13, record=True)
    assert t < 5000
    duals, zprev = [], np.zeros(p.m)
    for ww, zz, _ in hist:
        duals.append(oracle.srot_dual(ww, zprev, p.alpha, p.beta, p.C, reg))
        duals.append(oracle.srot_dual(ww, zz, p.alpha, p.beta, p.C, reg))
        zprev = zz
    assert all(b >= a - 1e-14 for a, b in zip(duals, duals[1:]))
    rep = oracle.srot_report(w, z, p.alpha, p.beta, p.C, reg)
    assert rep["row_l1"] < 1e-10 and rep["col_l1"] < 1e-12
    assert abs(rep["reg_primal"] - rep["dual"]) < 1e-10
    # the plan is sparse (squared regulariser: positive-part formula)
    T = oracle.srot_plan(w, z, p.C, reg)
    assert (T == 0).mean() > 0.3


def test_reduction_equals_explicit_problem():
    """Reduced C-SROT (2m dual variables) == SROT on the explicit d x d problem, by a generic solver."""
    p = synthetic.random_cyclic(seed=5, n=2, m=3)
    reg = ("squared", 0.8)
    w, z, _, _ = oracle.alternating_maximize(p.alpha, p.beta, p.C, reg, 20000, tol=1e-14)
    val = oracle.srot_report(w, z, p.alpha, p.beta, p.C, reg)["reg_primal"]
    a = oracle.expand_vector(p.alpha, p.n)
    b = oracle.expand_vector(p.beta, p.n)
    Cf = oracle.expand_cost(p.C)
    d = Cf.shape[0]
    obj = lambda x: float(Cf.ravel() @ x + (x * x).sum() / (2 * reg[1]))
    grad = lambda x: Cf.ravel() + x / reg[1]
    # the row and column constraints are dependent (both sum to 1): drop the last column constraint
    cons = [{"type": "eq", "fun": lambda x: x.reshape(d, d).sum(1) - a},
            {"type": "eq", "fun": lambda x: x.reshape(d, d).sum(0)[:-1] - b[:-1]}]
    res = scipy.optimize.minimize(obj, np.full(d * d, 1.0 / d ** 2), jac=grad, constraints=cons,
                                  bounds=[(0, None)] * (d * d), method="SLSQP",
                                  options={"ftol": 1e-15, "maxiter": 2000})
    assert res.success
    assert abs(res.fun - val) < 1e-8
