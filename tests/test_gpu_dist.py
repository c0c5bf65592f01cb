"""GPU tests of the row-sharded path on one B200.

Only one GPU is available, so ranks are emulated as shards held in one process: each shard runs
cerot_rows_shard on its rows, the column sums are summed on the device (the stand-in for ncclAllReduce), and
each shard applies cerot_zupdate. A real NCCL communicator of one rank exercises cerot_iter_sharded's
collective path end to end. Results are compared with the unsharded kernels and the oracle."""
import ctypes

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
        sh = cdist.ShardedCerot(_dev(p.C[:, b0:b0 + R, :]), _dev(p.alpha), _dev(p.beta), float(p.eps[0]), b0, p.m)
        out.append(sh.init())
    return out


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("maker", [lambda: synthetic.c2_ring(eps_factor=1e-2),
                                   lambda: synthetic.c4_large(m=256, n=16),
                                   lambda: synthetic.random_cyclic(seed=3, n=5, m=37, dtype=np.float32, eps=0.05)])
def test_emulated_row_sharding_matches_oracle(world, maker):
    p = maker()
    iters = 40
    shards = _shards(p, world)
    for sh in shards:   # the held rows of G are the rows of the unsharded G, bit for bit
        Go, Ao = oracle.aggregate(p.C)
        b0 = sh.row_begin
        assert np.array_equal(sh.G.cpu().numpy(), Go[b0:b0 + sh.R]) and np.array_equal(sh.argmin.cpu().numpy(),
                                                                                        Ao[b0:b0 + sh.R])
    for _ in range(iters):
        cs = [sh.rows().clone() for sh in shards]
        c = torch.stack(cs).sum(0)           # stand-in for the allreduce (rank order)
        for sh in shards:
            sh.zupdate(c)
    torch.cuda.synchronize()
    z0 = shards[0].z_hat.cpu().numpy()
    for sh in shards[1:]:
        assert np.array_equal(sh.z_hat.cpu().numpy(), z0)   # replicated q-update: bitwise identical
    w = np.zeros(p.m)
    for sh in shards:
        w[sh.row_begin:sh.row_begin + sh.R] = sh.w_hat.cpu().numpy()[sh.row_begin:sh.row_begin + sh.R]
    eps = float(p.eps[0])
    wo, zo, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, eps, iters, form="kernel")
    # gauge-invariant comparison: the plans agree (plan L1 within the parity bar)
    To = oracle.plan_blocks(wo, zo, p.C, eps)
    Tg = oracle.plan_blocks(w * eps, z0 * eps, p.C, eps)
    assert p.n * np.abs(Tg - To).sum() < 1e-5
    # plan rows of every shard == rows of the unsharded plan of the same potentials
    for sh in shards:
        T, _ = sh.plan(T_local=True)
        b0 = sh.row_begin
        ref = Tg[:, b0:b0 + sh.R, :]
        assert np.abs(T.cpu().numpy().astype(np.float64) - ref).max() <= 2e-7 * ref.max() + 1e-30


def test_sharded_expand_rows_bitexact():
    p = synthetic.random_cyclic(seed=8, n=4, m=24, dtype=np.float32, eps=0.1)
    blocks = np.random.default_rng(1).random((p.n, p.m, p.m)).astype(np.float32)
    full = oracle.expand_plan(blocks)
    for world in (2, 3):
        for r in range(world):
            b0, R = cdist.row_partition(p.m, world, r)
            sh = cdist.ShardedCerot(_dev(p.C[:, b0:b0 + R, :]), _dev(p.alpha), _dev(p.beta), 0.1, b0, p.m)
            rows = sh.expand(_dev(blocks[:, b0:b0 + R, :])).cpu().numpy()      # [n][R][d]
            for rr in range(p.n):
                assert np.array_equal(rows[rr], full[rr * p.m + b0: rr * p.m + b0 + R])


def test_nccl_single_rank_communicator():
    """cerot_iter_sharded / cerot_plan_sharded through a real NCCL communicator (1 rank): identical to the
    communicator-less path, and within the parity bar of the unsharded kernels."""
    L = cot.lib()
    uid = ctypes.create_string_buffer(128)
    assert L.cot_nccl_unique_id(uid) == 0, L.cot_last_error()
    comm = ctypes.c_void_p()
    assert L.cot_comm_init(uid, 1, 0, ctypes.byref(comm)) == 0, L.cot_last_error()

    class _C:
        handle = comm
    try:
        p = synthetic.c4_large(m=256, n=16)
        a = cdist.ShardedCerot(_dev(p.C), _dev(p.alpha), _dev(p.beta), float(p.eps[0]), 0, p.m, comm=_C()).init()
        b = cdist.ShardedCerot(_dev(p.C), _dev(p.alpha), _dev(p.beta), float(p.eps[0]), 0, p.m, comm=None).init()
        a.iterate(30)
        b.iterate(30)
        _, ra = a.plan()
        _, rb = b.plan()
        torch.cuda.synchronize()
        assert np.array_equal(a.z_hat.cpu().numpy(), b.z_hat.cpu().numpy())
        assert np.array_equal(ra.cpu().numpy(), rb.cpu().numpy())
        prob = cot.CerotProblem(_dev(p.C), _dev(p.alpha), _dev(p.beta), p.eps).init().iterate(30)
        _, rc = prob.plan()
        ga, gc = cdist.report_dict(ra), cot.report_dict(rc[0].cpu().numpy())
        assert abs(ga["objective"] - gc["objective"]) <= 1e-6 * abs(gc["objective"])
        assert abs(ga["dual"] - gc["dual"]) <= 1e-6 * abs(gc["dual"])
        assert abs(ga["row_l1"] - gc["row_l1"]) <= 1e-5
        it, conv, res = a.state()
        assert it == 30
    finally:
        L.cot_comm_destroy(comm)


@pytest.mark.parametrize("with_comm", [True, False], ids=["nccl1", "no_comm"])
def test_sharded_graph_replay_is_bitwise(with_comm, monkeypatch):
    """cerot_iter_sharded captures 8 iterations (row pass, column sums, allreduce, q-update) once as a CUDA
    graph and replays it; the tail runs as plain launches. Replay is the same work in the same order, so 37
    iterations (4 graph replays + 5 plain) and the freeze rule (tol > 0) are bit-identical to the per-iteration
    enqueue (COT_SHARDED_NO_GRAPH=1)."""
    L = cot.lib()
    comm = ctypes.c_void_p()
    if with_comm:
        uid = ctypes.create_string_buffer(128)
        assert L.cot_nccl_unique_id(uid) == 0, L.cot_last_error()
        assert L.cot_comm_init(uid, 1, 0, ctypes.byref(comm)) == 0, L.cot_last_error()

    class _C:
        handle = comm
    try:
        p = synthetic.c4_large(m=256, n=16)
        runs = []
        for no_graph in (False, True):
            if no_graph:
                monkeypatch.setenv("COT_SHARDED_NO_GRAPH", "1")
            else:
                monkeypatch.delenv("COT_SHARDED_NO_GRAPH", raising=False)
            a = cdist.ShardedCerot(_dev(p.C), _dev(p.alpha), _dev(p.beta), float(p.eps[0]), 0, p.m,
                                   comm=_C() if with_comm else None).init()
            a.iterate(37, tol=1e-6, check_every=4)
            torch.cuda.synchronize()
            runs.append((a.z_hat.cpu().numpy(), a.w_hat.cpu().numpy(), a.state()))
        (z0, w0, s0), (z1, w1, s1) = runs
        assert np.array_equal(z0, z1) and np.array_equal(w0, w1)
        assert s0 == s1
    finally:
        if with_comm:
            L.cot_comm_destroy(comm)


def test_batched_problem_sharding_is_exact():
    """C5 problem sharding: when every rank holds at least one problem per SM (the C5 regime: 4096 problems),
    a unit of rows is a whole problem, so solving a contiguous slice of the batch is bit-identical to the same
    problems inside the full batch (no data-path collective, no coupling). Smaller slices agree to rounding."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    p = synthetic.c5_batched(B=2 * sms, first=40)
    full = cot.CerotProblem(_dev(p.C), _dev(p.alpha), _dev(p.beta), _dev(p.eps)).init().iterate(20)
    _, rep_full = full.plan()
    world = 2
    for r in range(world):
        f, cnt = cdist.problem_partition(p.B, world, r)
        part = cot.CerotProblem(_dev(p.C[f:f + cnt]), _dev(p.alpha[f:f + cnt]), _dev(p.beta[f:f + cnt]),
                                _dev(p.eps[f:f + cnt])).init().iterate(20)
        _, rep = part.plan()
        assert np.array_equal(part.z_hat.cpu().numpy(), full.z_hat.cpu().numpy()[f:f + cnt])
        assert np.array_equal(rep.cpu().numpy(), rep_full.cpu().numpy()[f:f + cnt])
    q = synthetic.c5_batched(B=5, first=7)        # small slices: same results up to fp64 rounding
    fullq = cot.CerotProblem(_dev(q.C), _dev(q.alpha), _dev(q.beta), _dev(q.eps)).init().iterate(20)
    part = cot.CerotProblem(_dev(q.C[1:3]), _dev(q.alpha[1:3]), _dev(q.beta[1:3]), _dev(q.eps[1:3])).init().iterate(20)
    assert np.allclose(part.z_hat.cpu().numpy(), fullq.z_hat.cpu().numpy()[1:3], rtol=0, atol=1e-9)


def test_solve_sharded_single_rank_matches_solve():
    """cerot_solve_sharded (the whole solve of one rank) with a 1-rank NCCL communicator and without one:
    same iteration count and report as cerot_solve on the unsharded problem (C3, to tol 1e-8)."""
    L = cot.lib()
    uid = ctypes.create_string_buffer(128)
    assert L.cot_nccl_unique_id(uid) == 0, L.cot_last_error()
    comm = ctypes.c_void_p()
    assert L.cot_comm_init(uid, 1, 0, ctypes.byref(comm)) == 0, L.cot_last_error()

    class _C:
        handle = comm
    try:
        p = synthetic.c3_image(pair=2)
        _, _, _, reps = cot.cerot_solve(_dev(p.C), _dev(p.alpha), _dev(p.beta), p.eps, tol=1e-8, max_iter=3000,
                                        check_every=5)
        for c in (_C(), None):
            sh = cdist.ShardedCerot(_dev(p.C), _dev(p.alpha), _dev(p.beta), float(p.eps[0]), 0, p.m, comm=c)
            _, r = sh.solve(tol=1e-8, max_iter=3000, check_every=5)
            assert r["converged"] and r["iters"] == reps[0]["iters"]
            for k in ("objective", "dual"):
                assert abs(r[k] - reps[0][k]) <= 1e-6 * abs(reps[0][k])
    finally:
        L.cot_comm_destroy(comm)


def test_fused_over_nccl_symmetric_memory_single_rank():
    """The fused path's exchange buffers as NCCL symmetric memory (ncclMemAlloc + ncclCommWindowRegister, peer
    addresses from the window) instead of CUDA IPC: one rank, the same kernels; bitwise the same iterate as the
    IPC-mapped buffer (the exchange arithmetic does not depend on how the buffer was mapped)."""
    L = cot.lib()
    uid = ctypes.create_string_buffer(128)
    assert L.cot_nccl_unique_id(uid) == 0, L.cot_last_error()
    comm = ctypes.c_void_p()
    assert L.cot_comm_init(uid, 1, 0, ctypes.byref(comm)) == 0, L.cot_last_error()

    class _C:
        handle = comm
        rank = 0
        world = 1
    try:
        for maker in (lambda: synthetic.c4_large(m=512, n=16), lambda: synthetic.c4_large(m=1024, n=64)):
            p = maker()
            b0, R = cdist.row_partition(p.m, 8, 0) if p.n == 64 else (0, p.m)
            outs = []
            for kind in ("ipc", "ncclwin"):
                x = cdist.PeerExchange(p.m) if kind == "ipc" else cdist.NcclWindowExchange(p.m, _C())
                try:
                    sh = cdist.ShardedCerot(_dev(p.C[:, b0:b0 + R, :]), _dev(p.alpha), _dev(p.beta), float(p.eps[0]),
                                            b0, p.m).init()
                    sh.iterate_fused(x, 12)
                    sh.iterate_fused(x, 8)
                    torch.cuda.synchronize()
                    assert sh.state()[0] == 20
                    outs.append((sh.z_hat.cpu().numpy(), sh.w_hat.cpu().numpy()[b0:b0 + R]))
                finally:
                    x.close()
            assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    finally:
        L.cot_comm_destroy(comm)
