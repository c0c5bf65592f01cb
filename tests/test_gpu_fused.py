"""GPU tests of the fused row-sharded path: the exchange step of every iteration runs inside
the persistent kernel through LL lines in (peer-mapped) exchange buffers -- cerot_iter_fused.

One GPU is available, so the multi-rank protocol is tested the way B200_PROFILING.md prescribes: all ranks
of the partition run as ONE cooperative launch (cerot_iter_fused_emulated), each virtual rank on its own
slice of the SMs with its own shard, workspace, potentials and exchange buffer, spinning on the other
ranks' lines exactly as on separate GPUs. The per-GPU entry point (cerot_iter_fused through CUDA IPC
buffers, `PeerExchange`) runs here with one rank. Bars as tests/test_gpu_parity.py."""
import numpy as np
import pytest
import torch

import oracle
import synthetic

pytestmark = pytest.mark.gpu

cot = pytest.importorskip("paper_2311_13147_b200")
from paper_2311_13147_b200 import dist as cdist  # noqa: E402

DEV = torch.device("cuda:0")


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2311_13147_b200 import build
    build.build()
    cot.lib()


def _dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), device=DEV)


def _shards(p, world):
    out = []
    for r in range(world):
        b0, R = cdist.row_partition(p.m, world, r)
        out.append(cdist.ShardedCerot(_dev(p.C[:, b0:b0 + R, :]), _dev(p.alpha), _dev(p.beta), float(p.eps[0]), b0,
                                      p.m).init())
    return out


def _gather_w(shards, m):
    w = np.zeros(m)
    for sh in shards:
        w[sh.row_begin:sh.row_begin + sh.R] = sh.w_hat.cpu().numpy()[sh.row_begin:sh.row_begin + sh.R]
    return w


def _check_against_oracle(p, shards, iters):
    torch.cuda.synchronize()
    z0 = shards[0].z_hat.cpu().numpy()
    for sh in shards[1:]:   # the exchange sums in rank order on every rank: bitwise identical q-updates
        assert np.array_equal(sh.z_hat.cpu().numpy(), z0)
    eps = float(p.eps[0])
    w = _gather_w(shards, p.m)
    wo, zo, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, eps, iters, form="kernel")
    To = oracle.plan_blocks(wo, zo, p.C, eps)
    Tg = oracle.plan_blocks(w * eps, z0 * eps, p.C, eps)
    assert p.n * np.abs(Tg - To).sum() < 1e-5
    rg = oracle.report(w * eps, z0 * eps, p.alpha, p.beta, p.C, eps)
    ro = oracle.report(wo, zo, p.alpha, p.beta, p.C, eps)
    assert abs(rg["objective"] - ro["objective"]) <= 1e-6 * abs(ro["objective"])
    assert abs(rg["dual"] - ro["dual"]) <= 1e-6 * abs(ro["dual"])
    assert abs(rg["row_l1"] - ro["row_l1"]) <= 1e-5
    for sh in shards:
        it, conv, res = sh.state()
        assert it == iters


@pytest.mark.parametrize("kernel", ["res", "tma"])
@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("maker", [lambda: synthetic.c2_ring(eps_factor=1e-2),
                                   lambda: synthetic.c4_large(m=512, n=16),
                                   lambda: synthetic.c3_image()],
                         ids=["C2", "C4_m512_n16", "C3"])
def test_emulated_fused_matches_oracle(world, maker, kernel, monkeypatch):
    """Both per-rank kernels of the fused path: the on-chip-resident one (k_iter_res, where the shard fits) and the
    streaming one (k_iter_tma, COT_RES=0)."""
    if kernel == "tma":
        monkeypatch.setenv("COT_RES", "0")
    p = maker()
    iters = 30
    shards = _shards(p, world)
    xb = cdist.emulate_fused(shards, iters)
    try:
        _check_against_oracle(p, shards, iters)
    finally:
        cdist.free_xbufs(xb)


def test_emulated_fused_epoch_continues_across_calls():
    """Several launches on the same exchange buffers (the epoch keeps advancing; the two line slots are
    reused) == one launch of the summed count. Not bit for bit: each launch starts its row epilogues from
    the exact two-pass form (no previous row maximum), so the two differ by fp64 rounding only."""
    p = synthetic.c4_large(m=256, n=8)
    a = _shards(p, 4)
    b = _shards(p, 4)
    xa = cdist.emulate_fused(a, 7)
    for k in (1, 2, 4):
        cdist.emulate_fused(a, k, xbufs=xa)
    xb = cdist.emulate_fused(b, 14)
    torch.cuda.synchronize()
    try:
        for sa, sb in zip(a, b):
            for x, y in ((sa.z_hat, sb.z_hat), (sa.w_hat, sb.w_hat)):
                x, y = x.cpu().numpy(), y.cpu().numpy()
                assert np.abs(x - y).max() <= 1e-12 * max(1.0, np.abs(y).max()), np.abs(x - y).max()
        _check_against_oracle(p, a, 14)
    finally:
        cdist.free_xbufs(xa)
        cdist.free_xbufs(xb)


def test_emulated_fused_reinit_reuses_buffers():
    """cerot_init resets the solver state but not the exchange epoch: a second solve on the same buffers
    (after a 1-iteration solve, the case a state-derived generation would get wrong) matches a fresh one."""
    p = synthetic.c2_ring(eps_factor=1e-1)
    sh = _shards(p, 2)
    xb = cdist.emulate_fused(sh, 1)
    for s in sh:
        s.init()
    cdist.emulate_fused(sh, 9, xbufs=xb)
    try:
        _check_against_oracle(p, sh, 9)
    finally:
        cdist.free_xbufs(xb)


def test_emulated_fused_converges_like_the_oracle():
    """tol > 0: every virtual rank halts at the same iteration as the oracle's freeze rule."""
    p = synthetic.c3_image()
    eps = float(p.eps[0])
    tol = 1e-6
    shards = _shards(p, 3)
    xb = cdist.emulate_fused(shards, 400, tol=tol, check_every=1)
    torch.cuda.synchronize()
    try:
        its = [sh.state() for sh in shards]
        wo, zo, it_o, hist = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, eps, 400, tol=tol, check_every=1,
                                                    form="kernel", record=True)
        assert it_o < 400
        assert len({it for it, _, _ in its}) == 1
        it_g = its[0][0]
        for it, conv, res in its:
            assert conv == 1 and res <= tol
        if it_g != it_o:   # only where the fp64 monitor is within 1e-3 of tol at the deciding check
            assert abs(it_g - it_o) == 1
            assert abs(hist[min(it_g, it_o) - 1][2] / tol - 1) < 1e-3, (it_g, it_o)
        # the tol-run state against the oracle at the GPU's stopping iteration (plan, report, identical z_hat)
        _check_against_oracle(p, shards, it_g)
    finally:
        cdist.free_xbufs(xb)
    # and always at the oracle's stopping iteration: a fixed-count fused run of it_o iterations
    fixed = _shards(p, 3)
    xb = cdist.emulate_fused(fixed, it_o)
    try:
        _check_against_oracle(p, fixed, it_o)
    finally:
        cdist.free_xbufs(xb)


def test_fused_single_rank_ipc_buffer_matches_unsharded():
    """cerot_iter_fused (the per-GPU entry point, exchange buffer from cot_xchg_alloc) with one rank: the
    whole problem, the exchange with itself; agrees with the unsharded persistent kernel within the bar."""
    p = synthetic.c4_large(m=512, n=16)
    x = cdist.PeerExchange(p.m)
    try:
        sh = cdist.ShardedCerot(_dev(p.C), _dev(p.alpha), _dev(p.beta), float(p.eps[0]), 0, p.m).init()
        sh.iterate_fused(x, 12)
        sh.iterate_fused(x, 13)
        _, rep = sh.plan()
        prob = cot.CerotProblem(_dev(p.C), _dev(p.alpha), _dev(p.beta), p.eps).init().iterate(25)
        _, rc = prob.plan()
        torch.cuda.synchronize()
        g, c = cdist.report_dict(rep), cot.report_dict(rc[0].cpu().numpy())
        assert abs(g["objective"] - c["objective"]) <= 1e-6 * abs(c["objective"])
        assert abs(g["dual"] - c["dual"]) <= 1e-6 * abs(c["dual"])
        assert abs(g["row_l1"] - c["row_l1"]) <= 1e-5
        assert sh.state()[0] == 25
        _check_against_oracle(p, [sh], 25)
    finally:
        x.close()


def test_fused_argument_errors():
    p = synthetic.c2_ring()
    sh = _shards(p, 2)
    with pytest.raises(cot.CotError):   # unbalanced partition
        bad = cdist.ShardedCerot(_dev(p.C[:, :10, :]), _dev(p.alpha), _dev(p.beta), float(p.eps[0]), 0, p.m).init()
        cdist.emulate_fused([bad, sh[1]], 3)
    q = synthetic.random_cyclic(seed=2, n=3, m=30, dtype=np.float32, eps=0.1)   # m % 4 != 0
    with pytest.raises(cot.CotError):
        cdist.emulate_fused(_shards(q, 2), 3)


def test_emulated_fused_c4_full_size_8_ranks():
    """C4 (configs[3]) at full size (n = 64, m = 1024) split 8 ways -- the partition of the 8-GPU bench line --
    as 8 emulated ranks, 20 iterations, against the oracle (Alg. 2 with K precomputed, pinned equal to the
    streaming form)."""
    p = synthetic.c4_large()
    shards = _shards(p, 8)
    xb = cdist.emulate_fused(shards, 20)
    try:
        _check_against_oracle(p, shards, 20)
    finally:
        cdist.free_xbufs(xb)
