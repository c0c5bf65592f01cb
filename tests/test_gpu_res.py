"""GPU parity of K-ITER-RES (k_iter_res.cu), the on-chip-resident iteration kernel: the n*R*m costs of a problem
or row shard held in TMEM + shared memory of one CTA per SM, every Gibbs term re-evaluated each iteration, integer
column sums. Against the fp64 oracle (Alg. 2) with the bars of tests/test_gpu_parity.py,
through the C ABI; the shapes reach every layout branch: TMEM-only and TMEM + shared-memory quads, shared-memory
only (n > 64 or n % 4 != 0), the n % 8 == 4 tail of the TMEM k-loop, rows split over 2- and 4-CTA clusters
(DSMEM row exchange), ragged row ranges (R not a multiple of the cluster count), and the multi-GPU exchange level
(emulated ranks)."""
import math

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


def _check(p, prob, iters, obj_rtol=1e-6, l1_tol=1e-5):
    T, rep = prob.plan(T_blocks=True)
    torch.cuda.synchronize()
    it, _, _ = prob.state()
    assert it == iters
    eps = float(p.eps[0])
    w, z, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, eps, iters, form="kernel")
    ro = oracle.report(w, z, p.alpha, p.beta, p.C, eps)
    g = cot.report_dict(rep[0].cpu().numpy())
    for key in ("objective", "dual", "reg_primal"):
        assert math.isclose(g[key], ro[key], rel_tol=obj_rtol, abs_tol=1e-300), (key, g[key], ro[key])
    for key in ("row_l1", "col_l1"):
        assert abs(g[key] - ro[key]) <= l1_tol, (key, g[key], ro[key])
    To = oracle.plan_blocks(w, z, p.C, eps)
    assert p.n * np.abs(T.cpu().numpy().astype(np.float64) - To).sum() <= l1_tol
    # potentials (natural units) against the oracle's
    wg, zg = prob.w_hat.cpu().numpy() * eps, prob.z_hat.cpu().numpy() * eps
    # the potentials are defined up to a constant shift (w + c, z - c); compare the shift-invariant sums w_i + z_j
    d = (wg[:, None] + zg[None, :]) - (w[:, None] + z[None, :])
    assert np.abs(d).max() <= 1e-5 * max(1.0, np.abs(w).max()), np.abs(d).max()


def _problem(n, m, seed=11, eps_factor=0.05):
    rng = np.random.default_rng(seed)
    # points in the unit ball, n rotations about z (the C4 recipe at a smaller size)
    x = rng.normal(size=(m, 3))
    x /= np.maximum(1.0, np.linalg.norm(x, axis=1, keepdims=True))
    C = np.empty((n, m, m), np.float32)
    for k in range(n):
        a = 2 * np.pi * k / n
        Rz = np.array([[np.cos(a), -np.sin(a), 0], [np.sin(a), np.cos(a), 0], [0, 0, 1]])
        y = x @ Rz.T
        C[k] = ((x[:, None, :] - y[None, :, :]) ** 2).sum(-1)
    alpha = rng.dirichlet(np.ones(m)) / n
    beta = rng.dirichlet(np.ones(m)) / n
    eps = eps_factor * float(C.mean())
    return synthetic.Problem(name=f"res_n{n}_m{m}", C=C, alpha=alpha, beta=beta, eps=np.array([eps]), iters=60,
                             tol=0.0, meta={"seed": seed})


# (n, m, forced cluster size): TMEM-only quads (n = 64), TMEM + shared memory (n = 16 at m = 768: 1152 quads per
# CTA, 1024 in TMEM), shared memory only (n = 72 > 64; n = 6 not a multiple of 4), the n % 8 == 4 TMEM tail
# (n = 12), 2- and 4-CTA clusters (DSMEM row exchange) with ragged row ranges
_SHAPES = [(64, 256, 0), (16, 768, 0), (72, 256, 0), (6, 512, 0), (12, 512, 0), (16, 512, 2), (8, 1024, 4),
           (8, 768, 2), (24, 512, 4)]


@pytest.mark.parametrize("n,m,h", _SHAPES, ids=[f"n{n}_m{m}_h{h}" for n, m, h in _SHAPES])
def test_res_shapes_match_oracle(n, m, h, monkeypatch):
    if h:
        monkeypatch.setenv("COT_RES_H", str(h))
    p = _problem(n, m)
    assert cot.lib().cot_iter_path(1, n, m, 0, 0) == 4
    prob = cot.CerotProblem(_dev(p.C), _dev(p.alpha), _dev(p.beta), _dev(p.eps)).init()
    prob.iterate(40)
    prob.iterate(20)   # a second launch continues the first (sum buffers rotate by the workspace epoch)
    _check(p, prob, 60)


def test_res_reinit_and_solve_on_same_workspace():
    """cerot_init on a workspace the resident kernel already used (counters, sum slots) restarts cleanly."""
    p = synthetic.c3_image(pair=1)
    prob = cot.CerotProblem(_dev(p.C), _dev(p.alpha), _dev(p.beta), _dev(p.eps)).init()
    prob.iterate(7)
    prob.init().iterate(30)
    _check(p, prob, 30)


def test_res_eligibility():
    """Path selection: C3 and the 4-/8-way C4 shards are resident, C4 unsharded and the deterministic mode stream."""
    L = cot.lib()
    assert L.cot_iter_path(1, 4, 1024, 0, 0) == 4                  # C3
    assert L.cot_iter_path(1, 64, 1024, 0, 0) == 1                 # C4: 256 MB, streamed (k_iter_tma)
    assert L.cot_iter_path(1, 4, 1024, 0, 0x10) == 1               # COT_DETERMINISTIC: the streaming kernel
    assert L.cot_iter_path(1, 4, 1024, 0, 0x8) == 1                # COT_FORCE_TMA
    assert L.cot_iter_path(1, 4, 1000, 0, 0) == 1                  # m % 128 != 0
    assert L.cot_fused_path(64, 1024, 128, 8, 0, 0) == 4           # C4, 1 of 8 GPUs
    assert L.cot_fused_path(64, 1024, 512, 2, 0, 0) == 1           # C4, 1 of 2 GPUs: 128 MB per GPU, streamed
    assert L.cot_fused_path(64, 1024, 128, 8, 0, 0x10) == 1        # deterministic


@pytest.mark.parametrize("world", [2, 4])
def test_res_fused_emulated_ranks_match_oracle(world):
    """The multi-GPU exchange level of the resident kernel: `world` virtual ranks in one launch (1/world of the
    SMs each), rank-local integer sums pushed to every rank's exchange sums; bitwise identical z_hat on every
    rank (integer sums), and the oracle's iterate."""
    p = synthetic.c4_large(m=512, n=16)
    assert cot.lib().cot_fused_path(p.n, p.m, p.m // world, world, 1, 0) == 4
    shards = []
    for r in range(world):
        b0, R = cdist.row_partition(p.m, world, r)
        shards.append(cdist.ShardedCerot(_dev(p.C[:, b0:b0 + R, :]), _dev(p.alpha), _dev(p.beta), float(p.eps[0]),
                                         b0, p.m).init())
    xb = cdist.emulate_fused(shards, 25)
    try:
        cdist.emulate_fused(shards, 15, xbufs=xb)   # the exchange epoch continues across launches
        torch.cuda.synchronize()
        z0 = shards[0].z_hat.cpu().numpy()
        for sh in shards[1:]:
            assert np.array_equal(sh.z_hat.cpu().numpy(), z0)
        eps = float(p.eps[0])
        w = np.zeros(p.m)
        for sh in shards:
            w[sh.row_begin:sh.row_begin + sh.R] = sh.w_hat.cpu().numpy()[sh.row_begin:sh.row_begin + sh.R]
            assert sh.state()[0] == 40
        wo, zo, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, eps, 40, form="kernel")
        rg = oracle.report(w * eps, z0 * eps, p.alpha, p.beta, p.C, eps)
        ro = oracle.report(wo, zo, p.alpha, p.beta, p.C, eps)
        assert abs(rg["objective"] - ro["objective"]) <= 1e-6 * abs(ro["objective"])
        assert abs(rg["row_l1"] - ro["row_l1"]) <= 1e-5
        To = oracle.plan_blocks(wo, zo, p.C, eps)
        Tg = oracle.plan_blocks(w * eps, z0 * eps, p.C, eps)
        assert p.n * np.abs(Tg - To).sum() < 1e-5
    finally:
        cdist.free_xbufs(xb)


@pytest.mark.parametrize("ways", [8, 4], ids=["8_way_on_chip", "4_way_streamed_quads"])
def test_res_c4_shard_matches_streaming_kernel(ways):
    """C4 at full size (n = 64, m = 1024): rank 0's shard of the 8-way (128 rows, on chip) and of the 4-way partition
    (256 rows: ~13% of the quads streamed from L2 every iteration, k-split over four lanes) on the resident kernel
    with the exchange with itself (cerot_iter_fused, one rank) -- the per-GPU work of the 8- / 4-GPU runs -- gives
    the streaming kernel's iterate on the same shard (COT_RES=0; that kernel is pinned to the oracle by
    tests/test_gpu_fused.py) to fp32 k-sum rounding."""
    p = synthetic.c4_large()
    b0, R = cdist.row_partition(p.m, ways, 0)
    assert cot.lib().cot_fused_path(p.n, p.m, R, 1, 0, 0) == 4
    sh = cdist.ShardedCerot(_dev(p.C[:, b0:b0 + R, :]), _dev(p.alpha), _dev(p.beta), float(p.eps[0]), b0, p.m)
    x = cdist.PeerExchange(p.m)
    try:
        sh.init().iterate_fused(x, 20)
        torch.cuda.synchronize()
        assert sh.state()[0] == 20
        # the iterate of the fused path agrees with the streaming kernel on the same shard (COT_RES=0)
        import os
        os.environ["COT_RES"] = "0"
        try:
            sh2 = cdist.ShardedCerot(_dev(p.C[:, b0:b0 + R, :]), _dev(p.alpha), _dev(p.beta), float(p.eps[0]), b0, p.m)
            x2 = cdist.PeerExchange(p.m)
            sh2.init().iterate_fused(x2, 20)
            torch.cuda.synchronize()
            x2.close()
        finally:
            del os.environ["COT_RES"]
        z1, z2 = sh.z_hat.cpu().numpy(), sh2.z_hat.cpu().numpy()
        w1 = sh.w_hat.cpu().numpy()[b0:b0 + R]
        w2 = sh2.w_hat.cpu().numpy()[b0:b0 + R]
        assert np.abs(z1 - z2).max() <= 1e-6 * max(1.0, np.abs(z2).max()), np.abs(z1 - z2).max()
        assert np.abs(w1 - w2).max() <= 1e-6 * max(1.0, np.abs(w2).max()), np.abs(w1 - w2).max()
    finally:
        x.close()
