"""Pins for the oracle's structural functions (expand, symmetrize, aggregate, lift, fold).

Each check ties the oracle to something other than itself: SPEC/paper worked examples (tests/golden),
an independent construction (explicit d points -> d x d distance matrix; the permutation P of eq. A2),
or a property the definition implies (smallest argmin, G <= every C_k)."""
import numpy as np
import pytest

import oracle
import synthetic
from conftest import golden


# ---------------------------------------------------------------- expand (eq. blkstr_cost)
def test_expand_golden():
    g = golden("expand_examples.json")
    for case in g["cases"]:
        blocks = np.array(case["blocks"], dtype=np.float64)
        assert np.array_equal(oracle.expand_cost(blocks), np.array(case["dense"])), case["cite"]
        assert np.array_equal(oracle.expand_plan(blocks), np.array(case["dense"])), case["cite"]


def test_expand_plan_rows_golden_and_against_whole_plan():
    """expand_plan_rows (row sampling of Lemma 1's plan, for plans too large to build) on the SPEC worked
    examples (golden dense matrices) and, on random blocks, row for row against
    expand_plan -- including a broken placement that must be caught."""
    g = golden("expand_examples.json")
    for case in g["cases"]:
        blocks = np.array(case["blocks"], dtype=np.float64)
        dense = np.array(case["dense"])
        rows = list(range(dense.shape[0]))
        assert np.array_equal(oracle.expand_plan_rows(blocks, rows), dense), case["cite"]
    rng = np.random.default_rng(3)
    for n, m in [(1, 5), (3, 4), (7, 2)]:
        blocks = rng.random((n, m, m)).astype(np.float32)
        rows = rng.permutation(n * m)[: max(1, n * m // 2)]
        got = oracle.expand_plan_rows(blocks, rows)
        assert got.dtype == np.float32
        assert np.array_equal(got, oracle.expand_plan(blocks)[rows])
        if n > 1:   # a transposed shift (s + r instead of s - r) differs on some sampled row
            wrong = np.stack([np.concatenate([blocks[(s + I // m) % n][I % m] for s in range(n)]) for I in rows])
            assert not np.array_equal(got, wrong) or n == 2


def test_expand_vector_and_fold_golden():
    g = golden("expand_examples.json")
    for case in g["fold_average"]:
        assert np.allclose(oracle.fold_average(np.array(case["v"]), case["n"]), case["out"], atol=1e-15)
    a = np.array([0.1, 0.2, 0.3])
    assert np.array_equal(oracle.fold_average(oracle.expand_vector(a, 5), 5), a * 5 / 5)


def test_symmetrize_golden_and_properties():
    g = golden("expand_examples.json")
    for case in g["symmetrize"]:
        out = oracle.symmetrize(np.array(case["T"]), case["n"])
        assert np.allclose(out, case["out"], atol=1e-15), case["cite"]
    rng = np.random.default_rng(0)
    for n, m in [(2, 3), (3, 2), (4, 3), (6, 1)]:
        T = rng.random((n * m, n * m))
        S = oracle.symmetrize(T, n)
        assert np.allclose(oracle.symmetrize(S, n), S, atol=1e-14)          # idempotent
        assert np.isclose(S.sum(), T.sum(), rtol=1e-14)                      # mass preserved
        # S is block-circulant, so it equals the expansion of its first block row (eq. blkstr_optimal_solution)
        blocks = np.stack([S[0:m, s * m:(s + 1) * m] for s in range(n)])
        assert np.allclose(oracle.expand_plan(blocks), S, atol=1e-15)


def test_expand_is_fixed_point_of_shift():
    """Lemma 1's end of proof: P^l T (P^l)^T = T for a block-circulant T; the expansion
    (index-based) must satisfy it under the permutation of eq. A2 (matrix-based)."""
    rng = np.random.default_rng(1)
    for n, m in [(1, 4), (2, 3), (3, 3), (5, 2)]:
        blocks = rng.random((n, m, m))
        M = oracle.expand_cost(blocks)
        assert oracle.is_block_circulant(M, n)
        if n > 1:
            M2 = M.copy()
            M2[0, m] += 0.5                                                    # break one entry
            assert not oracle.is_block_circulant(M2, n)


@pytest.mark.parametrize("maker", [synthetic.c1_tiny, lambda: synthetic.c4_large(m=24, n=8)])
def test_expand_matches_explicit_point_cloud(maker):
    """Independent construction: the d points y_{s m + j} = R^s x_j, the d x d squared-distance matrix
    computed directly, must equal expand_cost of the generator's blocks (Assumption 1 holds)."""
    p = maker()
    n, m = p.n, p.m
    if "points" in p.meta:
        x = p.meta["points"]
        th = 2 * np.pi / n
        R = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
    else:
        rng = np.random.default_rng(p.meta["seed"])
        x = synthetic._unit_ball(rng, m)
        R = synthetic._rot3_z(2 * np.pi / n)
    pts = [x]
    for _ in range(n - 1):
        pts.append(pts[-1] @ R.T)
    Y = np.concatenate(pts)
    D = ((Y[:, None, :] - Y[None, :, :]) ** 2).sum(-1)
    E = oracle.expand_cost(p.C)
    tol = 1e-12 if p.C.dtype == np.float64 else 3e-6
    assert np.allclose(E, D, atol=tol, rtol=0)


def test_rotation_ordering_block_circulant():
    """SURVEY Q13 reading of P:194: the quadrant ordering makes the pixel-distance matrix exactly
    block-circulant (all even H <= 8, both metrics)."""
    for H in (2, 4, 6, 8):
        order = synthetic.rotation_quadrant_order(H)
        pix = order.reshape(-1, 2).astype(np.float64)
        assert len({tuple(p) for p in pix}) == H * H                     # a bijection onto the grid
        D = ((pix[:, None, :] - pix[None, :, :]) ** 2).sum(-1)
        assert oracle.is_block_circulant(D, 4)
        assert oracle.is_block_circulant(np.sqrt(D), 4)


def test_c3_generator_is_cyclic():
    p = synthetic.c3_image(H=16)
    order = synthetic.rotation_quadrant_order(16)
    pix = order.reshape(-1, 2).astype(np.float64)
    D = ((pix[:, None, :] - pix[None, :, :]) ** 2).sum(-1) / (2 * 15 ** 2)
    assert np.allclose(oracle.expand_cost(p.C), D.astype(np.float32), atol=0)
    assert np.isclose(p.alpha.sum(), 1 / 4) and np.isclose(p.beta.sum(), 1 / 4)
    assert (p.alpha > 0).all() and (p.beta > 0).all()


# ---------------------------------------------------------------- aggregate
def test_aggregate_golden():
    for case in golden("aggregate_examples.json")["cases"]:
        G, A = oracle.aggregate(np.array(case["C"], dtype=np.float64))
        assert np.array_equal(G, np.array(case["G"])), case["cite"]
        assert np.array_equal(A, np.array(case["A"])), case["cite"]


def test_aggregate_properties_with_ties():
    rng = np.random.default_rng(7)
    for trial in range(50):
        n, m = rng.integers(1, 7), rng.integers(1, 6)
        C = rng.integers(0, 3, size=(n, m, m)).astype(np.float64)         # many ties
        G, A = oracle.aggregate(C)
        for i in range(m):
            for j in range(m):
                col = C[:, i, j]
                assert G[i, j] == col.min()
                k = A[i, j]
                assert col[k] == col.min()
                assert all(col[kk] > col.min() for kk in range(k))         # the SMALLEST minimiser


def test_aggregate_signed_zero_and_batch():
    C = np.array([[[0.0]], [[-0.0]]])
    G, A = oracle.aggregate(C)
    assert A[0, 0] == 0 and not np.signbit(G[0, 0])
    C = np.array([[[-0.0]], [[0.0]]])
    G, A = oracle.aggregate(C)
    assert A[0, 0] == 0 and np.signbit(G[0, 0])
    rng = np.random.default_rng(3)
    Cb = rng.random((3, 4, 5, 5)).astype(np.float32)
    Gb, Ab = oracle.aggregate(Cb)
    for b in range(3):
        G1, A1 = oracle.aggregate(Cb[b])
        assert np.array_equal(Gb[b], G1) and np.array_equal(Ab[b], A1) and Gb.dtype == np.float32


# ---------------------------------------------------------------- lift
def test_lift_golden_and_mass():
    T = oracle.lift(np.array([[0.5]]), np.array([[1]]), 2)
    assert np.array_equal(T, np.array([[[0.0]], [[0.5]]]))
    rng = np.random.default_rng(2)
    S = rng.random((4, 4))
    S[1, 2] = 0.0
    A = rng.integers(0, 3, size=(4, 4))
    T = oracle.lift(S, A, 3)
    assert np.array_equal(T.sum(0), S)                                     # sum_k T_k = S exactly
    assert (T[:, 1, 2] == 0).all()
    assert np.array_equal(oracle.lift(S, np.zeros((4, 4), int), 1)[0], S)  # S:217 (n = 1)


def test_c2_sweep_is_configs1():
    """bench.py's C2 workload = BASELINE configs[1] as stated: the ring problem at eps in {1e-1, 1e-2, 1e-3} x
    mean(C), as one batch of three independent problems sharing C, alpha and beta (each problem equal to the
    single-eps generator's)."""
    p = synthetic.c2_sweep()
    assert p.batched and p.B == 3 and p.n == 8 and p.m == 128 and p.iters == 500 and p.C.dtype == np.float32
    for b, f in enumerate((1e-1, 1e-2, 1e-3)):
        q = synthetic.c2_ring(eps_factor=f)
        assert np.array_equal(p.C[b], q.C) and np.array_equal(p.alpha[b], q.alpha) and np.array_equal(p.beta[b], q.beta)
        assert p.eps[b] == q.eps[0]
        assert np.isclose(p.eps[b], f * p.C[b].astype(np.float64).mean(), rtol=1e-12)
