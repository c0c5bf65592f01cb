"""NEXT-4: the host network simplex for the small LOT (clot_small_lot in libcyclicot, host C++; no GPU).
Pinned against the oracle's LP (HiGHS on the same problem, oracle.lot) and the paper-fixed facts: the SPEC
worked examples (tests/golden/lot_examples.json), the LP optimality certificate (dual feasibility
and complementary slackness, the phi = 0 case of eq. optimality_condition), vertex solutions
(at most 2m-1 non-zeros), Theorem 1 through Alg. 1 (value n <G, S*> = the full d x d LP)."""
import numpy as np
import pytest

import oracle
import synthetic
from paper_2311_13147_b200 import build as _build
from paper_2311_13147_b200 import host_lp
from conftest import golden


@pytest.fixture(scope="module", autouse=True)
def _lib():
    _build.build()


def _check_certificate(alpha, beta, G, S, u, v, tol=1e-9):
    scale = max(1.0, np.abs(G).max())
    assert S.min() >= 0.0
    assert np.abs(S.sum(1) - alpha).max() <= 1e-12 * max(1.0, alpha.sum()) + 1e-15
    assert np.abs(S.sum(0) - beta).max() <= 1e-12 * max(1.0, beta.sum()) + 1e-15
    red = G - u[:, None] - v[None, :]
    assert red.min() >= -tol * scale                       # dual feasibility
    assert np.abs(red[S > 0]).max() <= tol * scale         # complementary slackness
    assert (S > 0).sum() <= 2 * len(alpha) - 1             # a vertex of the transportation polytope


def test_spec_worked_examples():
    for ex in golden("lot_examples.json")["small_lot"]:
        a, b, G = (np.array(ex[k], dtype=np.float64) for k in ("alpha", "beta", "G"))
        val, S, u, v, _ = host_lp.small_lot(a, b, G, duals=True)
        assert abs(val - ex["value"]) <= 1e-12, ex["cite"]
        assert np.allclose(S, np.array(ex["S"]), atol=1e-12), ex["cite"]
        _check_certificate(a, b, G, S, u, v)


@pytest.mark.parametrize("seed", range(200))
def test_random_small_instances_match_the_lp(seed):
    rng = np.random.default_rng(seed)
    m = int(rng.integers(1, 9))
    a = rng.dirichlet(np.ones(m))
    b = rng.dirichlet(np.ones(m))
    G = rng.integers(0, 4, size=(m, m)).astype(np.float64) if seed % 2 else rng.random((m, m))   # ties when even
    val, S, u, v, _ = host_lp.small_lot(a, b, G, duals=True)
    ref, _ = oracle.lot(a, b, G)
    assert abs(val - ref) <= 1e-9
    _check_certificate(a, b, G, S, u, v)


def test_degenerate_uniform_permutation_costs():
    m = 16
    perm = np.random.default_rng(3).permutation(m)
    G = np.ones((m, m))
    G[np.arange(m), perm] = 0.0
    a = np.full(m, 1.0 / m)
    val, S, u, v, _ = host_lp.small_lot(a, a, G, duals=True)
    assert val == 0.0
    assert np.allclose(S[np.arange(m), perm], 1.0 / m)
    _check_certificate(a, a, G, S, u, v)


def test_scaling_invariance_and_negative_costs():
    rng = np.random.default_rng(11)
    m = 12
    a, b = rng.dirichlet(np.ones(m)), rng.dirichlet(np.ones(m))
    G = rng.random((m, m))
    v1, _ = host_lp.small_lot(a, b, G)
    v2, _ = host_lp.small_lot(a, b, 7.5 * G)
    v3, _ = host_lp.small_lot(a, b, G - 3.0)          # shifting costs shifts the value by -3 * mass
    assert abs(v2 - 7.5 * v1) <= 1e-12 * 7.5
    assert abs(v3 - (v1 - 3.0)) <= 1e-12


@pytest.mark.parametrize("maker", [lambda: synthetic.c1_tiny(), lambda: synthetic.c5_batched(B=1, first=3)],
                         ids=["C1", "C5_problem3"])
def test_config_instances_match_the_lp_and_theorem1(maker):
    p = maker()
    C = p.C[0] if p.C.ndim == 4 else p.C
    alpha = p.alpha[0] if p.alpha.ndim == 2 else p.alpha
    beta = p.beta[0] if p.beta.ndim == 2 else p.beta
    G, A = oracle.aggregate(C)
    val, S, u, v, piv = host_lp.small_lot(alpha, beta, G, duals=True)
    ref, _ = oracle.lot(alpha, beta, G)
    assert abs(val - ref) <= 1e-9 * max(1.0, abs(ref))
    _check_certificate(alpha, beta, G.astype(np.float64), S, u, v)
    if C.shape[0] * C.shape[1] <= 64:   # Theorem 1: n <G, S*> equals the full d x d LP
        full, _ = oracle.lot_full(alpha, beta, C)
        assert abs(C.shape[0] * val - full) <= 1e-9


def test_argument_errors():
    from paper_2311_13147_b200 import CotError
    with pytest.raises(CotError):
        host_lp.small_lot(np.array([0.5, 0.5]), np.array([0.9, 0.3]), np.zeros((2, 2)))   # unequal mass
    with pytest.raises(CotError):
        host_lp.small_lot(np.array([1.0, 0.0]), np.array([0.5, 0.5]), np.zeros((2, 2)))   # zero entry
    with pytest.raises(CotError):
        host_lp.small_lot(np.array([1.0]), np.array([1.0]), np.array([[np.nan]]))


def test_clot_lot_value_applies_full_scale_factor():
    """clot_lot_value: the library returns the explicit problem's C-LOT value n * <G, S*> (Theorem 1)
    -- equal to the oracle's brute-force LP on the expanded d x d problem (C1)."""
    import ctypes
    import oracle
    import synthetic
    import paper_2311_13147_b200 as cot
    p = synthetic.c1_tiny()
    G, _ = oracle.aggregate(p.C)
    m = p.m
    S = np.zeros((m, m))
    full, small = ctypes.c_double(), ctypes.c_double()
    a, b, Gc = (np.ascontiguousarray(x, dtype=np.float64) for x in (p.alpha, p.beta, G))
    assert cot.lib().clot_lot_value(a.ctypes.data_as(ctypes.c_void_p), b.ctypes.data_as(ctypes.c_void_p),
                                    Gc.ctypes.data_as(ctypes.c_void_p), m, p.n, S.ctypes.data_as(ctypes.c_void_p),
                                    ctypes.byref(full), ctypes.byref(small)) == 0
    assert abs(full.value - p.n * small.value) <= 1e-15 * abs(full.value)
    ref, _ = oracle.lot(oracle.expand_vector(p.alpha, p.n), oracle.expand_vector(p.beta, p.n),
                        oracle.expand_cost(p.C))
    assert abs(full.value - ref) <= 1e-9 * max(1.0, abs(ref))
    assert cot.lib().clot_lot_value(None, None, None, m, 0, None, ctypes.byref(full), None) == -1
