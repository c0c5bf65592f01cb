"""Multi-GPU drivers, one process per GPU, torch.distributed for the plumbing.

* Row sharding of one large problem (C4): rank g holds rows [row_begin, row_begin + R) of every cost block;
  the p-update of those rows is local, the plan column sums are summed across ranks with ONE m-length fp64
  ncclAllReduce per iteration (issued by libcyclicot on the compute stream, through a library-owned NCCL
  communicator), and every rank applies the identical q-update. `ShardedCerot`.
* Problem sharding of a batch (C5): independent problems are split across ranks with no data-path
  collective. `problem_partition`.

The communicator is bootstrapped through torch.distributed: rank 0 creates the 128-byte ncclUniqueId with
cot_nccl_unique_id, it is broadcast as a uint8 tensor, and every rank calls cot_comm_init.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Tuple

import numpy as np

from . import (COT_COLD_START, REPORT_FIELDS, _check, _dtype_code, _ptr, _stream, lib)

__all__ = ["row_partition", "problem_partition", "broadcast_bytes", "NcclComm", "ShardedCerot"]


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

    def expand(self, T_local, out=None):
        """The held rows of the dense d x d plan: [n][R][d] (row (r, i) = full row r*m + row_begin + i)."""
        import torch
        d = self.n * self.m
        out = torch.empty((self.n, self.R, d), dtype=T_local.dtype, device=T_local.device) if out is None else out
        _check(lib().clot_expand_shard(_ptr(T_local), None, self.n, self.R, self.m, self.dt, _ptr(out),
                                       _stream(self.stream)), "clot_expand_shard")
        return out

    def state(self):
        it = (ctypes.c_int64 * 1)()
        cv = (ctypes.c_int32 * 1)()
        rs = (ctypes.c_double * 1)()
        _check(lib().cerot_state(_ptr(self.ws), 1, self.m, self.n, self.dt, it, cv, rs, _stream(self.stream)),
               "cerot_state")
        return int(it[0]), int(cv[0]), float(rs[0])


def report_dict(rep) -> dict:
    v = [float(x) for x in np.asarray(rep.cpu() if hasattr(rep, "cpu") else rep).reshape(-1)]
    return dict(zip(REPORT_FIELDS, v))
