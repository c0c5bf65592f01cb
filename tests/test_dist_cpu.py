"""CPU tests of the multi-GPU host logic (gloo, world_size 2): row / problem partitioning, the byte broadcast
that bootstraps the NCCL communicator, and the row-sharded decomposition the library implements
(local p-update of the held rows -> local plan column sums -> allreduce -> identical q-update on every rank),
checked against the unsharded oracle iteration. The per-rank compute here is the oracle's arithmetic written
per row (test code); on the GPU the same steps are cerot_rows_shard / ncclAllReduce / cerot_zupdate."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synthetic
from paper_2311_13147_b200 import dist as cdist


def test_partitions_cover_exactly_and_balance():
    for m in (1, 7, 128, 1024, 1000):
        for world in (1, 2, 3, 4, 8):
            if world > m:
                continue
            spans = [cdist.row_partition(m, world, r) for r in range(world)]
            rows = [i for b, R in spans for i in range(b, b + R)]
            assert rows == list(range(m))
            assert max(R for _, R in spans) - min(R for _, R in spans) <= 1
    for B in (1, 5, 4096):
        for world in (1, 2, 3, 8):
            spans = [cdist.problem_partition(B, world, r) for r in range(world)]
            probs = [i for f, c in spans for i in range(f, f + c)]
            assert probs == list(range(B))
    with pytest.raises(ValueError):
        cdist.row_partition(2, 3, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # 1) the communicator bootstrap: a 128-byte id from rank 0 reaches every rank unchanged
        payload = bytes(range(128)) if rank == 0 else None
        got = cdist.broadcast_bytes(payload, 128, 0)
        assert got == bytes(range(128))
        # 2) the row-sharded iteration, eps-scaled potentials as in the library (w_hat = w/eps)
        p = synthetic.random_cyclic(seed=42, n=5, m=13, eps=0.07)
        eps = float(p.eps[0])
        C = p.C.astype(np.float64)
        b0, R = cdist.row_partition(p.m, world, rank)
        rows = slice(b0, b0 + R)
        zh = np.zeros(p.m)
        wh = np.zeros(p.m)
        for _ in range(25):
            # p-update of the held rows: w_i = log alpha_i - log sum_{j,k} exp(z_j - C_ijk/eps)
            X = zh[None, None, :] - C[:, rows, :] / eps
            mx = X.max(axis=(0, 2))
            wh_loc = np.log(p.alpha[rows]) - mx - np.log(np.exp(X - mx[None, :, None]).sum(axis=(0, 2)))
            # local plan column sums c_j = sum_{i held, k} exp(w_i + z_j - C_ijk/eps)
            c_loc = np.exp(wh_loc[None, :, None] + X).sum(axis=(0, 1))
            c = torch.from_numpy(c_loc.copy())
            dist.all_reduce(c)                                   # the one exchange step per iteration
            zh = zh + np.log(p.beta) - np.log(c.numpy())         # identical q-update on every rank
            wh[:] = 0.0
            wh[rows] = wh_loc
        w_all = torch.from_numpy(wh.copy())
        dist.all_reduce(w_all)
        out[rank] = (zh, w_all.numpy())
    finally:
        dist.destroy_process_group()


def test_row_sharded_decomposition_gloo():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    p = synthetic.random_cyclic(seed=42, n=5, m=13, eps=0.07)
    eps = float(p.eps[0])
    w, z, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, eps, 25)
    for r in range(world):
        zh, wh = out[r]
        assert np.abs(zh * eps - z).max() < 1e-12       # z replicated and equal to the unsharded iterate
        assert np.abs(wh * eps - w).max() < 1e-12       # union of the held rows' w = the unsharded w
    assert np.array_equal(out[0][0], out[1][0])         # bitwise identical q-updates on both ranks


def _worker_fused(rank, world, port, out):
    """Host logic of the fused path (cerot_iter_fused): the 64-byte IPC handles travel with allgather_bytes;
    each rank's column sums reach every rank (the kernel's peer stores; all_gather here) and are summed in
    RANK ORDER on every rank, so the q-updates are bitwise identical although the data are split unevenly."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        handles = cdist.allgather_bytes(bytes([rank]) * 64)
        assert handles == [bytes([q]) * 64 for q in range(world)]
        p = synthetic.random_cyclic(seed=7, n=4, m=20, eps=0.05)
        eps = float(p.eps[0])
        C = p.C.astype(np.float64)
        b0, R = cdist.row_partition(p.m, world, rank)
        assert R in (p.m // world, -(-p.m // world))       # the balanced partition cerot_iter_fused requires
        rows = slice(b0, b0 + R)
        zh = np.zeros(p.m)
        for _ in range(20):
            X = zh[None, None, :] - C[:, rows, :] / eps
            mx = X.max(axis=(0, 2))
            wh_loc = np.log(p.alpha[rows]) - mx - np.log(np.exp(X - mx[None, :, None]).sum(axis=(0, 2)))
            c_loc = torch.from_numpy(np.exp(wh_loc[None, :, None] + X).sum(axis=(0, 1)))
            lines = [torch.empty_like(c_loc) for _ in range(world)]
            dist.all_gather(lines, c_loc)                       # every rank's lines of every slice
            c = np.zeros(p.m)
            for q in range(world):                              # rank order, as the kernel sums them
                c = c + lines[q].numpy()
            zh = zh + np.log(p.beta) - np.log(c)
        out[rank] = zh
    finally:
        dist.destroy_process_group()


def test_fused_exchange_rank_order_gloo():
    world = 3
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_fused, args=(world, port, out), nprocs=world, join=True)
    p = synthetic.random_cyclic(seed=7, n=4, m=20, eps=0.05)
    _, z, _, _ = oracle.cyclic_sinkhorn(p.alpha, p.beta, p.C, float(p.eps[0]), 20)
    for r in range(world):
        assert np.array_equal(out[r], out[0])                  # bitwise identical on every rank
    assert np.abs(out[0] * float(p.eps[0]) - z).max() < 1e-12
