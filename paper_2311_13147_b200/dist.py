"""Multi-GPU drivers, one process per GPU, torch.distributed for the plumbing.

* Row sharding of one large problem (C4): rank g holds rows [row_begin, row_begin + R) of every cost block;
  the p-update of those rows is local, the plan column sums are summed across ranks with ONE m-length fp64
  ncclAllReduce per iteration (issued by libcyclicot on the compute stream, through a library-owned NCCL
  communicator), and every rank applies the identical q-update. `ShardedCerot`.
* Problem sharding of a batch (C5): independent problems are split across ranks with no data-path
  collective. `problem_partition`.

The communicator is bootstrapped through torch.distributed: rank 0 creates the 128-byte ncclUniqueId with
cot_nccl_unique_id, it is broadcast as a uint8 tensor, and every rank calls cot_comm_init.

* Fused row sharding (the default multi-GPU path of bench.py): the same partition and arithmetic, but the
  exchange step runs inside the persistent iteration kernel (cerot_iter_fused): each rank's column sums are
  written straight into every rank's exchange buffer over NVLink (CUDA IPC peer mappings set up once by
  `PeerExchange`; the 64-byte handles travel through torch.distributed) and summed in rank order on every
  rank. `emulate_fused` runs all ranks' fused iterations as one cooperative launch on one GPU (the test
  harness of the protocol when fewer GPUs than ranks are available).
"""
from __future__ import annotations

import ctypes
from typing import Optional, Tuple

import numpy as np

from . import (COT_COLD_START, REPORT_FIELDS, _check, _dtype_code, _ptr, _stream, lib)

__all__ = ["row_partition", "problem_partition", "broadcast_bytes", "allgather_bytes", "NcclComm",
           "PeerExchange", "ShardedCerot", "emulate_fused"]


def row_partition(m: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced split of the m rows: rank r gets [row_begin, row_begin + R)."""
    if not (0 <= rank < world) or m < world:
        raise ValueError("need 0 <= rank < world <= m")
    base, rem = divmod(m, world)
    begin = rank * base + min(rank, rem)
    return begin, base + (1 if rank < rem else 0)


def problem_partition(B: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced split of B independent problems: (first, count)."""
    base, rem = divmod(B, world)
    first = rank * base + min(rank, rem)
    return first, base + (1 if rank < rem else 0)


def broadcast_bytes(payload: Optional[bytes], nbytes: int, src: int = 0, group=None, device=None) -> bytes:
    """Broadcast `nbytes` raw bytes from rank `src` through torch.distributed (works with gloo and nccl)."""
    import torch
    import torch.distributed as dist
    t = torch.zeros(nbytes, dtype=torch.uint8, device=device or "cpu")
    if dist.get_rank(group) == src:
        t.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    dist.broadcast(t, src=src, group=group)
    return bytes(t.cpu().numpy().tobytes())


def allgather_bytes(payload: bytes, group=None, device=None) -> list:
    """Every rank's `payload` (same length on every rank), in rank order (gloo or nccl)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.frombuffer(bytearray(payload), dtype=torch.uint8).to(device or "cpu")
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return [bytes(o.cpu().numpy().tobytes()) for o in out]


class PeerExchange:
    """This rank's exchange buffer of the fused path plus every other rank's, mapped with CUDA IPC.

    xbufs is the HOST array of device pointers cerot_iter_fused takes: entry q = rank q's buffer as
    addressed by this process (entry `rank` = the local buffer). Collective: every rank constructs it."""

    def __init__(self, m: int, group=None):
        import torch
        import torch.distributed as dist
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.local = ctypes.c_void_p()
        handle = ctypes.create_string_buffer(64)
        _check(lib().cot_xchg_alloc(m, self.world, ctypes.byref(self.local), handle), "cot_xchg_alloc")
        self.opened = []
        ptrs = [None] * self.world
        ptrs[self.rank] = self.local.value
        if self.world > 1:
            dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else None
            handles = allgather_bytes(handle.raw, group, dev)
            for q, h in enumerate(handles):
                if q == self.rank:
                    continue
                pq = ctypes.c_void_p()
                _check(lib().cot_xchg_open(ctypes.create_string_buffer(h, 64), ctypes.byref(pq)), "cot_xchg_open")
                self.opened.append(pq)
                ptrs[q] = pq.value
        self.xbufs = (ctypes.c_void_p * self.world)(*ptrs)

    def close(self):
        for pq in self.opened:
            lib().cot_xchg_close(pq)
        self.opened = []
        if self.local:
            lib().cot_xchg_free(self.local)
            self.local = ctypes.c_void_p()


class NcclWindowExchange:
    """The fused path's exchange buffers as NCCL symmetric memory (ncclMemAlloc + ncclCommWindowRegister) instead
    of CUDA IPC handles: the same cerot_iter_fused kernels, the peer addresses taken from the NCCL window. For
    processes that cannot share CUDA IPC handles. Collective: every rank constructs (and closes) it."""

    def __init__(self, m: int, comm: "NcclComm"):
        self.comm = comm
        self.world = comm.world
        self.rank = comm.rank
        self.local = ctypes.c_void_p()
        self.win = ctypes.c_void_p()
        _check(lib().cot_xchg_nccl_alloc(comm.handle, m, self.world, ctypes.byref(self.local), ctypes.byref(self.win)),
               "cot_xchg_nccl_alloc")
        self.xbufs = (ctypes.c_void_p * self.world)()
        _check(lib().cot_xchg_nccl_peers(self.win, self.world, self.xbufs), "cot_xchg_nccl_peers")

    def close(self):
        if self.local:
            lib().cot_xchg_nccl_free(self.comm.handle, self.local, self.win)
            self.local = ctypes.c_void_p()


class NcclComm:
    """A libcyclicot-owned NCCL communicator over all ranks of the default torch.distributed group."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        uid = None
        if self.rank == 0:
            buf = ctypes.create_string_buffer(128)
            _check(lib().cot_nccl_unique_id(buf), "cot_nccl_unique_id")
            uid = buf.raw
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else None
        uid = broadcast_bytes(uid, 128, 0, group, dev)
        self._id = ctypes.create_string_buffer(uid, 128)
        self.handle = ctypes.c_void_p()
        _check(lib().cot_comm_init(self._id, self.world, self.rank, ctypes.byref(self.handle)), "cot_comm_init")

    def close(self):
        if self.handle:
            lib().cot_comm_destroy(self.handle)
            self.handle = ctypes.c_void_p()


class ShardedCerot:
    """Rows [row_begin, row_begin + R) of one C-EROT problem on this GPU (row sharding).

    C_local: device [n][R][m] (the held rows of every block); alpha, beta: full [m] fp64; eps scalar.
    comm: NcclComm (None = single GPU / emulation: the caller reduces the column sums itself)."""

    def __init__(self, C_local, alpha, beta, eps, row_begin: int, m: int, comm: Optional[NcclComm] = None,
                 stream=None):
        import torch
        self.C = C_local
        self.n, self.R, m2 = C_local.shape
        assert m2 == m
        self.m, self.row_begin = m, row_begin
        self.dt = _dtype_code(C_local)
        dev = C_local.device
        self.alpha = alpha.to(torch.float64).contiguous()
        self.beta = beta.to(torch.float64).contiguous()
        self.eps = torch.as_tensor(eps, dtype=torch.float64, device=dev).reshape(1).contiguous()
        self.w_hat = torch.zeros(m, dtype=torch.float64, device=dev)
        self.z_hat = torch.zeros(m, dtype=torch.float64, device=dev)
        self.comm = comm
        self.stream = stream
        nbytes = int(lib().cot_workspace_bytes_sharded(self.n, m, self.R, self.dt))
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self.G = torch.empty((self.R, m), dtype=C_local.dtype, device=dev)
        self.argmin = torch.empty((self.R, m), dtype=torch.int32, device=dev)
        self.c_local = torch.empty(m, dtype=torch.float64, device=dev)
        nf = torch.zeros(1, dtype=torch.int32, device=dev)
        s = _stream(stream)
        _check(lib().clot_aggregate_shard(_ptr(C_local), self.n, self.R, m, self.dt, _ptr(self.G), _ptr(self.argmin),
                                          _ptr(nf), s), "clot_aggregate_shard")
        _check(lib().cot_check_nonfinite(_ptr(nf), s), "clot_aggregate_shard")

    @property
    def _comm(self):
        return self.comm.handle if self.comm is not None else None

    def init(self, cold: bool = True):
        _check(lib().cerot_init(_ptr(self.alpha), _ptr(self.beta), 1, self.m, COT_COLD_START if cold else 0,
                                _ptr(self.z_hat), _ptr(self.ws), self.ws.numel(), _stream(self.stream)), "cerot_init")
        return self

    def iterate(self, iters: int, tol: float = 0.0, check_every: int = 1, flags: int = 0):
        _check(lib().cerot_iter_sharded(_ptr(self.alpha), _ptr(self.beta), _ptr(self.C), _ptr(self.G), self.n, self.m,
                                        self.row_begin, self.R, self.dt, _ptr(self.eps), iters, tol, check_every,
                                        flags, _ptr(self.w_hat), _ptr(self.z_hat), _ptr(self.ws), self.ws.numel(),
                                        self._comm, _stream(self.stream)), "cerot_iter_sharded")
        return self

    def solve(self, tol: float = 0.0, max_iter: int = 1000, check_every: int = 1, T_local: bool = False):
        """The whole solve of this rank (cerot_solve_sharded): returns (T_local or None, report dict)."""
        import torch
        from . import cot_report, STATUS
        T = torch.empty_like(self.C) if T_local else None
        rep = cot_report()
        code = lib().cerot_solve_sharded(_ptr(self.alpha), _ptr(self.beta), _ptr(self.C), self.n, self.m,
                                         self.row_begin, self.R, self.dt, _ptr(self.eps), tol, max_iter, check_every,
                                         COT_COLD_START, _ptr(self.w_hat), _ptr(self.z_hat), _ptr(T), _ptr(self.ws),
                                         self.ws.numel(), self._comm, ctypes.byref(rep), _stream(self.stream))
        _check(code, "cerot_solve_sharded", ok=(0, 1))
        d = {f: getattr(rep, f) for f in REPORT_FIELDS}
        d.update(iters=rep.iters, converged=bool(rep.converged), status=STATUS[rep.status])
        return T, d

    def iterate_fused(self, xchg: "PeerExchange", iters: int, tol: float = 0.0, check_every: int = 1,
                      flags: int = 0):
        """`iters` iterations with the exchange inside the persistent kernel (cerot_iter_fused)."""
        _check(lib().cerot_iter_fused(_ptr(self.alpha), _ptr(self.beta), _ptr(self.C), _ptr(self.G), self.n, self.m,
                                      self.row_begin, self.R, self.dt, _ptr(self.eps), iters, tol, check_every, flags,
                                      _ptr(self.w_hat), _ptr(self.z_hat), _ptr(self.ws), self.ws.numel(), xchg.world,
                                      xchg.rank, xchg.xbufs, _stream(self.stream)), "cerot_iter_fused")
        return self

    # the two halves, for callers that reduce the column sums themselves (emulation, tests)
    def rows(self, flags: int = 0):
        _check(lib().cerot_rows_shard(_ptr(self.alpha), _ptr(self.C), _ptr(self.G), self.n, self.m, self.row_begin,
                                      self.R, self.dt, _ptr(self.eps), flags, _ptr(self.z_hat), _ptr(self.w_hat),
                                      _ptr(self.c_local), _ptr(self.ws), self.ws.numel(), _stream(self.stream)),
               "cerot_rows_shard")
        return self.c_local

    def zupdate(self, c, tol: float = 0.0, check_every: int = 1):
        _check(lib().cerot_zupdate(_ptr(self.beta), _ptr(c), self.n, self.m, tol, check_every, _ptr(self.z_hat),
                                   _ptr(self.ws), self.ws.numel(), _stream(self.stream)), "cerot_zupdate")

    def plan(self, T_local: bool = False):
        """Plan of the held rows (T_local [n][R][m]) and the report reduced over all ranks."""
        import torch
        T = torch.empty_like(self.C) if T_local else None
        rep = torch.empty(8, dtype=torch.float64, device=self.C.device)
        _check(lib().cerot_plan_sharded(_ptr(self.alpha), _ptr(self.beta), _ptr(self.C), _ptr(self.G), self.n, self.m,
                                        self.row_begin, self.R, self.dt, _ptr(self.eps), _ptr(self.w_hat),
                                        _ptr(self.z_hat), _ptr(T), _ptr(rep), _ptr(self.ws), self.ws.numel(),
                                        self._comm, _stream(self.stream)), "cerot_plan_sharded")
        return T, rep

    def expand(self, T_local, out=None, argmin=None):
        """The held rows of the dense d x d plan: [n][R][d] (row (r, i) = full row r*m + row_begin + i).
        T_local: C-EROT blocks [n][R][m], or with argmin [R][m] (C-LOT lift) the small-LP solution rows S [R][m]."""
        import torch
        d = self.n * self.m
        out = torch.empty((self.n, self.R, d), dtype=T_local.dtype, device=T_local.device) if out is None else out
        _check(lib().clot_expand_shard(_ptr(T_local), _ptr(argmin), self.n, self.R, self.m, self.dt, _ptr(out),
                                       _stream(self.stream)), "clot_expand_shard")
        return out

    def state(self):
        it = (ctypes.c_int64 * 1)()
        cv = (ctypes.c_int32 * 1)()
        rs = (ctypes.c_double * 1)()
        _check(lib().cerot_state(_ptr(self.ws), 1, self.m, self.n, self.dt, it, cv, rs, _stream(self.stream)),
               "cerot_state")
        return int(it[0]), int(cv[0]), float(rs[0])


def emulate_fused(shards, iters: int, tol: float = 0.0, check_every: int = 1, flags: int = 0, xbufs=None,
                  stream=None):
    """All ranks' fused iterations in ONE cooperative launch on one GPU (cerot_iter_fused_emulated).

    shards: list of ShardedCerot (rank order, one device, balanced partition). xbufs: per-rank exchange
    buffers from cot_xchg_alloc (allocated here when None; returned so that later calls reuse them -- the
    epoch inside each buffer must keep advancing)."""
    V = len(shards)
    L = lib()
    if xbufs is None:
        xbufs = []
        for _ in range(V):
            b = ctypes.c_void_p()
            _check(L.cot_xchg_alloc(shards[0].m, V, ctypes.byref(b), None), "cot_xchg_alloc")
            xbufs.append(b.value)
    P = ctypes.c_void_p
    arr = lambda xs: (P * V)(*xs)
    s0 = shards[0]
    _check(L.cerot_iter_fused_emulated(
        V, _ptr(s0.alpha), _ptr(s0.beta), arr([_ptr(s.C) for s in shards]), arr([_ptr(s.G) for s in shards]),
        s0.n, s0.m, (ctypes.c_int64 * V)(*[s.row_begin for s in shards]), (ctypes.c_int64 * V)(*[s.R for s in shards]),
        s0.dt, _ptr(s0.eps), iters, tol, check_every, flags, arr([_ptr(s.w_hat) for s in shards]),
        arr([_ptr(s.z_hat) for s in shards]), arr([_ptr(s.ws) for s in shards]),
        (ctypes.c_size_t * V)(*[s.ws.numel() for s in shards]), arr(xbufs), _stream(stream)),
        "cerot_iter_fused_emulated")
    return xbufs


def free_xbufs(xbufs):
    for b in xbufs or []:
        lib().cot_xchg_free(b)


def report_dict(rep) -> dict:
    v = [float(x) for x in np.asarray(rep.cpu() if hasattr(rep, "cpu") else rep).reshape(-1)]
    return dict(zip(REPORT_FIELDS, v))
