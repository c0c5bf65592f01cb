"""Pins for the oracle's LOT side: the plain LP (HiGHS), Algorithm 1 and Theorem 1.

Pins: SPEC worked examples (golden), the closed form of the 2 x 2 transportation polytope (one free
parameter, optimum at an endpoint), Theorem 1's value equality against the brute-force LP on the explicit
d x d problem (random tiny instances), the App. A counter-example values, and the divisor
invariance of P:595."""
import math

import numpy as np
import pytest

import oracle
import synthetic
from conftest import golden


def test_small_lot_golden():
    for case in golden("lot_examples.json")["small_lot"]:
        v, S = oracle.lot(np.array(case["alpha"]), np.array(case["beta"]), np.array(case["G"], float))
        assert abs(v - case["value"]) <= 1e-12, case["cite"]
        assert np.allclose(S, case["S"], atol=1e-12), case["cite"]


def test_lot_2x2_closed_form():
    """2 x 2 transportation polytope: S00 = t, S01 = a0 - t, S10 = b0 - t, S11 = a1 - b0 + t with
    t in [max(0, b0 - a1), min(a0, b0)]; the objective is linear in t, so the LP value is the smaller
    of the two endpoint values (an independent solution of the same LP)."""
    rng = np.random.default_rng(11)
    for _ in range(100):
        a = rng.dirichlet([1, 1])
        b = rng.dirichlet([1, 1])
        G = rng.random((2, 2)) * 3
        lo, hi = max(0.0, b[0] - a[1]), min(a[0], b[0])
        f = lambda t: G[0, 0] * t + G[0, 1] * (a[0] - t) + G[1, 0] * (b[0] - t) + G[1, 1] * (a[1] - b[0] + t)
        expect = min(f(lo), f(hi))
        v, S = oracle.lot(a, b, G)
        assert abs(v - expect) <= 1e-10
        assert np.allclose(S.sum(1), a, atol=1e-10) and np.allclose(S.sum(0), b, atol=1e-10)


def test_clot_golden_and_naive_strategy():
    for case in golden("lot_examples.json")["clot"]:
        C = np.array(case["C"], dtype=np.float64)
        r = oracle.clot(np.array(case["alpha"]), np.array(case["beta"]), C)
        assert abs(r["value"] - case["value"]) <= 1e-12, case["cite"]
        assert np.allclose(r["T_blocks"], case["T_blocks"], atol=1e-12)
        vfull, _ = oracle.lot_full(np.array(case["alpha"]), np.array(case["beta"]), C)
        assert abs(vfull - case["value"]) <= 1e-12
        assert abs(oracle.naive_tile_lot(np.array(case["alpha"]), np.array(case["beta"]), C)
                   - case["naive_value"]) <= 1e-12


def test_theorem1_random_tiny_instances():
    """Theorem 1: n * (small LOT on G) == LOT on the explicit d x d problem, and the lifted,
    expanded plan is feasible with that cost. 200 instances, m <= 8, n <= 4."""
    rng = np.random.default_rng(1234)
    for t in range(200):
        n = int(rng.integers(2, 5))
        m = int(rng.integers(2, 9))
        p = synthetic.random_cyclic(seed=10_000 + t, n=n, m=m, integer=bool(t % 3 == 0))
        r = oracle.clot(p.alpha, p.beta, p.C)
        vfull, _ = oracle.lot_full(p.alpha, p.beta, p.C)
        assert abs(r["value"] - vfull) <= 1e-9, (t, r["value"], vfull)
        Tfull = oracle.expand_plan(r["T_blocks"])
        a = oracle.expand_vector(p.alpha, n)
        b = oracle.expand_vector(p.beta, n)
        assert np.abs(Tfull.sum(1) - a).max() <= 1e-10 and np.abs(Tfull.sum(0) - b).max() <= 1e-10
        assert abs((oracle.expand_cost(p.C) * Tfull).sum() - vfull) <= 1e-9
        # complementary support: T_k > 0 only where C_k == G
        G = r["G"]
        for k in range(n):
            assert np.all((r["T_blocks"][k] <= 0) | (p.C[k] == G))


def test_c1_clot_equals_full_lp():
    """C1 (configs[0], d = 64): the reduction equals the brute-force LP on the explicit problem."""
    p = synthetic.c1_tiny()
    r = oracle.clot(p.alpha, p.beta, p.C)
    vfull, _ = oracle.lot_full(p.alpha, p.beta, p.C)
    assert abs(r["value"] - vfull) <= 1e-12 * max(1.0, vfull) + 1e-13


@pytest.mark.parametrize("metric", ["euclidean", "squared"])
def test_counter_example(metric):
    """App. A: the cyclic reduction gives the true optimum (1.0); solving one component and
    tiling gives sqrt(2) (Euclidean) / 2.0 (squared)."""
    g = golden("counter_example.json")[metric]
    p = synthetic.counter_example(metric)
    r = oracle.clot(p.alpha, p.beta, p.C)
    # the explicit problem has zero-mass pixels: alpha, beta contain zeros; the LP handles them
    vfull, _ = oracle.lot_full(p.alpha, p.beta, p.C)
    assert abs(vfull - g["full_lp_value"]) <= 1e-9
    assert abs(r["value"] - g["full_lp_value"]) <= 1e-9
    naive = oracle.naive_tile_lot(p.alpha, p.beta, p.C)
    assert abs(naive - g["naive_tile_value"]) <= 1e-9
    assert naive > r["value"] + 0.4


def test_divisor_invariance_lot():
    """data symmetric at order n_max is symmetric at every divisor n; every n gives the same
    C-LOT value. The order-n blocks are read off the explicit matrix (block row 0 at block size d/n)."""
    p = synthetic.appd_synthetic(seed=0, d=24, n_max=6)
    a = oracle.expand_vector(p.alpha, 6)
    b = oracle.expand_vector(p.beta, 6)
    Cfull = oracle.expand_cost(p.C)
    vals = []
    for n in (1, 2, 3, 6):
        m = 24 // n
        blocks = np.stack([Cfull[0:m, s * m:(s + 1) * m] for s in range(n)])
        assert np.array_equal(oracle.expand_cost(blocks), Cfull)
        vals.append(oracle.clot(a[:m], b[:m], blocks)["value"])
    assert max(vals) - min(vals) <= 1e-9
