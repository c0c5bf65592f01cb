"""GPU tests of the deterministic mode (COT_DETERMINISTIC; SURVEY §8(e) "bitwise identical for G = 1, 2, 4, 8").

Column partials are accumulated exactly in 128-bit fixed point and every row's statistics in a fixed warp
order, so the iterates must not depend on the row partition: the unsharded persistent kernel on all SMs, on
fewer SMs, and 2/4/8 emulated ranks of the fused path (one cooperative launch, each virtual rank on 1/N of the
SMs: the profiling recipe's way of testing ranks that wait on each other on one GPU) give bitwise identical
potentials, and stay within the parity bars of the oracle; a solve split over several launches reproduces one launch
bit for bit."""
import os

import numpy as np
import pytest
import torch

import oracle
import synthetic

pytestmark = pytest.mark.gpu

cot = pytest.importorskip("paper_2311_13147_b200")
from paper_2311_13147_b200 import dist as cdist  # noqa: E402

DEV = torch.device("cuda:0")
DET = cot.COT_DETERMINISTIC


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2311_13147_b200 import build
    build.build()
    cot.lib()


def _dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), device=DEV)


def _unsharded(p, iters_list, max_ctas=None):
    old = os.environ.get("COT_MAX_CTAS")
    if max_ctas:
        os.environ["COT_MAX_CTAS"] = str(max_ctas)
    try:
        prob = cot.CerotProblem(_dev(p.C), _dev(p.alpha), _dev(p.beta), _dev(p.eps)).init()
        for k in iters_list:
            prob.iterate(k, flags=DET)
        torch.cuda.synchronize()
        return prob.w_hat.cpu().numpy(), prob.z_hat.cpu().numpy()
    finally:
        if max_ctas:
            if old is None:
                del os.environ["COT_MAX_CTAS"]
            else:
                os.environ["COT_MAX_CTAS"] = old


def _emulated(p, world, iters):
    shards = []
    for r in range(world):
        b0, R = cdist.row_partition(p.m, world, r)
        shards.append(cdist.ShardedCerot(_dev(p.C[:, b0:b0 + R, :]), _dev(p.alpha), _dev(p.beta), float(p.eps[0]),
                                         b0, p.m).init())
    xb = cdist.emulate_fused(shards, iters, flags=DET)
    torch.cuda.synchronize()
    try:
        w = np.zeros(p.m)
        for sh in shards:
            w[sh.row_begin:sh.row_begin + sh.R] = sh.w_hat.cpu().numpy()[sh.row_begin:sh.row_begin + sh.R]
        zs = [sh.z_hat.cpu().numpy() for sh in shards]
        return w, zs
    finally:
        cdist.free_xbufs(xb)


@pytest.mark.parametrize("maker", [lambda: synthetic.c4_large(m=512, n=16), lambda: synthetic.c3_image(),
                                   lambda: synthetic.c4_large()], ids=["C4_m512_n16", "C3", "C4_full"])
def test_bitwise_identical_across_partitions(maker):
    p = maker()
    iters = 25
    w1, z1 = _unsharded(p, [iters])
    # fewer SMs (other rows per CTA): same bits
    w2, z2 = _unsharded(p, [iters], max_ctas=128)
    assert np.array_equal(w1.view(np.uint64), w2.view(np.uint64))
    assert np.array_equal(z1.view(np.uint64), z2.view(np.uint64))
    for world in (2, 4, 8):
        w, zs = _emulated(p, world, iters)
        for z in zs:
            assert np.array_equal(z.view(np.uint64), z1.view(np.uint64)), world
        assert np.array_equal(w.view(np.uint64), w1.view(np.uint64)), world
    # and within the parity bars of the oracle
    eps = float(p.eps[0])
    wo, zo, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, eps, iters, form="kernel")
    rg = oracle.report(w1 * eps, z1 * eps, p.alpha, p.beta, p.C, eps)
    ro = oracle.report(wo, zo, p.alpha, p.beta, p.C, eps)
    assert abs(rg["objective"] - ro["objective"]) <= 1e-6 * abs(ro["objective"])
    assert abs(rg["dual"] - ro["dual"]) <= 1e-6 * abs(ro["dual"])
    assert abs(rg["row_l1"] - ro["row_l1"]) <= 1e-5


def test_fixed_point_range_is_enforced():
    """The 128-bit fixed point has 8 integer bits: a problem with sum(alpha) >= 2^7 (un-normalised masses) is
    refused by the deterministic launch (COT_E_ARG at the state check), not silently wrapped; the same problem
    runs in the default mode and matches the oracle (the solver itself is scale-agnostic)."""
    p = synthetic.c4_large(m=256, n=8)
    scale = 200.0 * p.n            # sum(alpha) = 200
    a, b = p.alpha * scale, p.beta * scale
    prob = cot.CerotProblem(_dev(p.C), _dev(a), _dev(b), _dev(p.eps)).init()
    prob.iterate(5, flags=DET)
    with pytest.raises(cot.CotError) as e:
        prob.state()
    assert e.value.code == -1 and "2^7" in str(e.value)
    prob2 = cot.CerotProblem(_dev(p.C), _dev(a), _dev(b), _dev(p.eps)).init()
    prob2.iterate(5)
    it, _, _ = prob2.state()
    assert it[0] == 5
    eps = float(p.eps[0])
    wo, zo, _, _ = oracle.cyclic_sinkhorn(a, b, p.C, eps, 5, form="kernel")
    w, z = prob2.w_hat.cpu().numpy(), prob2.z_hat.cpu().numpy()
    rg = oracle.report(w * eps, z * eps, a, b, p.C, eps)
    ro = oracle.report(wo, zo, a, b, p.C, eps)
    assert abs(rg["objective"] - ro["objective"]) <= 1e-6 * abs(ro["objective"])


def test_split_entry_points_reject_deterministic():
    """cerot_rows / the NCCL sharded path have no fixed-point partials: COT_DETERMINISTIC is an argument error
    with an explicit message (not an opaque CUDA 'invalid argument')."""
    p = synthetic.c4_large(m=256, n=8)
    sh = cdist.ShardedCerot(_dev(p.C), _dev(p.alpha), _dev(p.beta), float(p.eps[0]), 0, p.m).init()
    with pytest.raises(cot.CotError) as e:
        sh.iterate(2, flags=DET)
    assert e.value.code == -1 and "COT_DETERMINISTIC" in str(e.value)


@pytest.mark.parametrize("maker", [lambda: synthetic.c4_large(m=512, n=16), lambda: synthetic.c3_image()],
                         ids=["C4_m512_n16", "C3"])
def test_bitwise_identical_across_launch_boundaries(maker):
    """COT_DETERMINISTIC: the row shift is the exact maximum every iteration and the column sums are exact, so a
    solve split over several launches (7 + 11 + 7) gives the bits of one 25-iteration launch."""
    p = maker()
    w1, z1 = _unsharded(p, [25])
    for split in ([7, 11, 7], [1, 23, 1], [12, 13]):   # 1-iteration launches keep no k-blocks resident
        w2, z2 = _unsharded(p, split)
        assert np.array_equal(z1.view(np.uint64), z2.view(np.uint64)), split
        assert np.array_equal(w1.view(np.uint64), w2.view(np.uint64)), split
