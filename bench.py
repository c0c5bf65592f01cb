#!/usr/bin/env python
"""bench.py — throughput of the C-EROT hot path (BASELINE.json metric) on B200, plus the oracle baseline.

A "step" is one pass of the whole hot path over one synthetic problem whose
inputs are already resident in HBM:
    clot_aggregate (G, argmin) -> cerot_init (validation, q = 1) -> `iters` cyclic Sinkhorn iterations
    (cerot_rows + cerot_cols each) -> cerot_plan (T blocks + fp64 report) -> clot_expand (dense d x d plan)
value = Gibbs-kernel evaluations (n * m^2 * iters * B) / device time of the step (whole job, all ranks).

Default workload: C4 (BASELINE.json configs[3]: n = 64, m = 1024, d = 65536, fp32, eps = 5e-3, 500
iterations), the largest single-GPU configuration the metric is quoted on ("% of HBM roofline").

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--workload C4|C2|C3|C5]
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

DEFAULT_METRIC = "C-EROT Gibbs-kernel evals/s (n·m² per iter) and % of HBM/SFU roofline, 1–8 GPU"
UNIT = "Gibbs-kernel evals/s"
_JSON_OUT = sys.stdout   # replaced in main() by the saved stdout


def _metric() -> str:
    try:
        with open(os.path.join(ROOT, "BASELINE.json")) as f:
            return json.load(f)["metric"]
    except Exception:
        return DEFAULT_METRIC


def _peaks():
    """Roofline denominators: MEASURED_PEAKS.json (driver-written) else the profiling guide's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _ncu_traffic_per_iter(workload: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per iteration of the dominant kernel, from the committed
    ncu --set full summary (profiles/ncu_summary.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        return d.get(workload, {}).get("dram_bytes_per_iteration")
    except Exception:
        return None


# ------------------------------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock + throttle reasons with NVML during the timed region (B200_PROFILING.md)."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, local_rank: int):
        self.samples, self.reasons, self.ok = [], 0, False
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            idx = local_rank
            parts = [x for x in vis.split(",") if x.strip()]
            if parts and all(x.strip().isdigit() for x in parts):
                idx = int(parts[local_rank])
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------ workloads
def make_problem(workload: str, iters_override: int | None):
    import synthetic
    if workload == "C4":
        p = synthetic.c4_large()
    elif workload == "C2":   # configs[1]: the three eps values of the sweep, one batch of independent problems
        p = synthetic.c2_sweep()
    elif workload == "C2e2":   # a single C2 problem (eps = 1e-2 * mean C): the latency-bound case
        p = synthetic.c2_ring(eps_factor=1e-2)
    elif workload == "C3":
        p = synthetic.c3_image()
    elif workload == "C5":
        p = synthetic.c5_batched(B=int(os.environ.get("COT_C5_B", "4096")))
    else:
        raise SystemExit(f"unknown workload {workload}")
    iters = iters_override or p.iters
    return p, iters


# ------------------------------------------------------------------------------------------ our arm
class Runner:
    """Device-resident buffers and one step of the hot path through the C ABI (raw ctypes calls)."""

    def __init__(self, p, iters, dev, stream, sample_every=10):
        import torch
        import paper_2311_13147_b200 as cot
        self.cot, self.L, self.torch = cot, cot.lib(), torch
        self.p, self.iters, self.dev, self.stream = p, iters, dev, stream
        self.B, self.n, self.m = p.B, p.n, p.m
        self.dt = cot.COT_F32 if p.C.dtype == np.float32 else cot.COT_F64
        self.C = torch.as_tensor(np.ascontiguousarray(p.C), device=dev)
        self.alpha = torch.as_tensor(np.ascontiguousarray(p.alpha), device=dev)
        self.beta = torch.as_tensor(np.ascontiguousarray(p.beta), device=dev)
        self.eps = torch.as_tensor(np.ascontiguousarray(p.eps), device=dev)
        shp = (self.B, self.m, self.m)
        self.G = torch.empty(shp, dtype=self.C.dtype, device=dev)
        self.A = torch.empty(shp, dtype=torch.int32, device=dev)
        self.w = torch.zeros_like(self.alpha)
        self.z = torch.zeros_like(self.beta)
        self.ws = cot.workspace(self.B, self.n, self.m, self.dt, dev)
        self.Tb = torch.empty_like(self.C)
        d = self.n * self.m
        self.Tfull = torch.empty((self.B, d, d), dtype=self.C.dtype, device=dev)
        self.rep = torch.empty((self.B, 8), dtype=torch.float64, device=dev)
        self.sample_every = sample_every
        self.ev = []       # (start, end) events around sampled row-pass launches
        self.s = stream.cuda_stream
        P = lambda t: t.data_ptr()
        self.ptr = dict(C=P(self.C), a=P(self.alpha), b=P(self.beta), e=P(self.eps), G=P(self.G), A=P(self.A),
                        w=P(self.w), z=P(self.z), ws=P(self.ws), Tb=P(self.Tb), Tf=P(self.Tfull), rep=P(self.rep))
        self.flags = int(os.environ.get("COT_BENCH_FLAGS", "0"), 0)
        self.pre = os.environ.get("COT_BENCH_MODE") == "precomputed"   # NEXT-1 line (separate metric)
        self.S = torch.empty((self.B, 1, self.m, self.m), dtype=self.C.dtype, device=dev) if self.pre else None
        # which iteration kernel the library runs: 1 = persistent TMA stream (all iterations in one launch),
        # 2 = cluster-resident (all iterations in one launch, whole problems on chip), 0 = launch pair / iteration
        self.path = int(self.L.cot_iter_path(self.B, 1 if self.pre else self.n, self.m, self.dt, self.flags))
        self.persistent = self.path in (1, 2, 3, 4)
        self.launches_per_step = 1 + 1 + (1 if self.persistent else 2 * iters) + 3 + 1 + (1 if self.pre else 0)
        self.bytes_iter = float(p.B) * ((2 if self.pre else p.n + 1) * p.m * p.m) * p.C.itemsize

    def _ck(self, code, fn):
        if code != 0:
            raise RuntimeError(f"{fn} failed ({code}): {self.L.cot_last_error().decode()}")

    def step(self, record=False, C_ptr=None):
        L, q, s = self.L, dict(self.ptr), self.s
        if C_ptr is not None:   # e2e pipelining: this step's cost blocks live in another device buffer
            q["C"] = C_ptr
        B, n, m, dt = self.B, self.n, self.m, self.dt
        wsn = self.ws.numel()
        self._ck(L.clot_aggregate(q["C"], B, n, m, dt, q["G"], q["A"], None, s), "clot_aggregate")
        self._ck(L.cerot_init(q["a"], q["b"], B, m, 1, q["z"], q["ws"], wsn, s), "cerot_init")
        if record:
            e0 = self.torch.cuda.Event(enable_timing=True)
            e1 = self.torch.cuda.Event(enable_timing=True)
            e0.record(self.stream)
        if self.pre:   # NEXT-1: S once, then O(m^2) iterations on (S, G)
            self._ck(L.cerot_precompute(q["C"], q["G"], B, n, m, dt, q["e"], self.S.data_ptr(), s), "cerot_precompute")
            self._ck(L.cerot_iter(q["a"], q["b"], self.S.data_ptr(), q["G"], B, 1, m, dt, q["e"], self.iters, 0.0, 1,
                                  self.flags | 4, q["w"], q["z"], q["ws"], wsn, s), "cerot_iter")
        else:
            self._ck(L.cerot_iter(q["a"], q["b"], q["C"], q["G"], B, n, m, dt, q["e"], self.iters, 0.0, 1, self.flags,
                                  q["w"], q["z"], q["ws"], wsn, s), "cerot_iter")
        if record:
            e1.record(self.stream)
            self.ev.append((e0, e1))
        self._ck(L.cerot_plan(q["a"], q["b"], q["C"], q["G"], B, n, m, dt, q["e"], q["w"], q["z"], q["Tb"], q["rep"],
                              q["ws"], wsn, s), "cerot_plan")
        self._ck(L.clot_expand(q["Tb"], None, B, n, m, dt, q["Tf"], s), "clot_expand")

    def input_bytes(self):
        """Device bytes the step reads as input (the cost blocks dominate)."""
        return self.C.numel() * self.C.element_size() + 2 * self.alpha.numel() * 8

    def iter_kernel_ms(self):
        """Device time of the iteration launch(es) of each timed step (CUDA events on our stream)."""
        ts = [a.elapsed_time(b) for a, b in self.ev]
        return statistics.mean(ts), statistics.median(ts), len(ts)

    def report_row(self):
        return self.rep.cpu().numpy()[0]

    def e2e_inputs(self):
        return self.p.C, self.C, [(self.p.alpha, self.alpha), (self.p.beta, self.beta), (self.p.eps, self.eps)], \
            [self.rep, self.w, self.z]


class stdout_to_stderr:
    """Route the process's C-level stdout to stderr (NCCL prints its version banner at communicator init);
    bench.py's stdout carries exactly one JSON line."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *a):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


class ShardedRunner:
    """Row sharding of one problem over the ranks: this rank holds rows
    [row_begin, row_begin + R) of every block; one fp64 ncclAllReduce of the m column sums per iteration
    inside libcyclicot (cerot_iter_sharded); plan report reduced across ranks; each rank expands its rows."""

    def __init__(self, p, iters, dev, stream, rank, world):
        import torch
        import paper_2311_13147_b200 as cot
        from paper_2311_13147_b200 import dist as cdist
        assert not p.batched
        self.cot, self.cdist, self.L, self.torch = cot, cdist, cot.lib(), torch
        self.p, self.iters, self.stream = p, iters, stream
        self.B, self.n, self.m = 1, p.n, p.m
        self.row_begin, self.R = cdist.row_partition(p.m, world, rank)
        # fused (default): the exchange inside the persistent kernel over peer-mapped buffers (cerot_iter_fused),
        # mapped with CUDA IPC, else (IPC refused, or its probe failed) as NCCL symmetric memory (the same kernel
        # over ncclCommWindowRegister'ed buffers); COT_SHARD_IMPL=ncclwin: only the latter; COT_SHARD_IMPL=nccl:
        # the baseline, one ncclAllReduce + 3 launches per iteration (cerot_iter_sharded)
        impl = os.environ.get("COT_SHARD_IMPL", "fused")
        kinds = {"fused": ["ipc", "ncclwin"], "ncclwin": ["ncclwin"]}.get(impl, [])
        self.flags = int(os.environ.get("COT_BENCH_FLAGS", "0"), 0)   # e.g. 0x10: COT_DETERMINISTIC
        self.fused_note = None
        import torch.distributed as tdist

        def agree(ok):   # every rank must take the same path
            flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
            if tdist.is_initialized():
                tdist.all_reduce(flag, op=tdist.ReduceOp.MIN)
            return int(flag.item()) == 1
        with stdout_to_stderr():
            self.comm = cdist.NcclComm()
        self.xchg = None
        Cl = np.ascontiguousarray(p.C[:, self.row_begin:self.row_begin + self.R, :])
        self.Cl_host = Cl
        self.sh = cdist.ShardedCerot(torch.as_tensor(Cl, device=dev), torch.as_tensor(p.alpha, device=dev),
                                     torch.as_tensor(p.beta, device=dev), float(p.eps[0]), self.row_begin, p.m,
                                     comm=self.comm, stream=stream)
        self.xkind, notes = None, []
        for kind in kinds:
            ok, err = True, ""
            try:
                with stdout_to_stderr():
                    self.xchg = cdist.PeerExchange(p.m) if kind == "ipc" else cdist.NcclWindowExchange(p.m, self.comm)
            except Exception as e:   # e.g. IPC not permitted in this container, no NCCL symmetric memory
                ok, err = False, str(e)
            if agree(ok):
                # probe: a few fused iterations must complete on every rank (peer stores visible, no COT_E_PEER)
                try:
                    with stdout_to_stderr():
                        self.sh.init().iterate_fused(self.xchg, 3)
                        if self.sh.state()[0] != 3:
                            ok, err = False, "probe iterations incomplete"
                except Exception as e:
                    ok, err = False, str(e)
                if agree(ok):
                    self.xkind = kind
                    break
                err = "probe failed: " + (err or "on another rank")
            if self.xchg is not None:
                self.xchg.close()
                self.xchg = None
            notes.append(f"{kind}: {err or 'unavailable on another rank'}")
            print(f"[bench] fused exchange over {kind} not used ({notes[-1]})", file=sys.stderr)
        self.fused = self.xkind is not None
        if not self.fused and kinds:
            self.fused_note = "fused exchange unavailable (" + "; ".join(notes) + "): NCCL baseline"
        # flags actually run: the NCCL baseline has no fixed-point partials (COT_DETERMINISTIC is the fused path's)
        self.flags_requested = self.flags
        if not self.fused and self.flags & 0x10:
            self.flags &= ~0x10
            self.fused_note = (self.fused_note or "NCCL baseline") + "; COT_DETERMINISTIC dropped (fused path only)"
        self.exchange = {"path": ("fused" + ("" if self.xkind == "ipc" else " (NCCL symmetric memory)")) if self.fused
                         else "nccl",
                         "probe": ("ok (3 fused iterations on every rank" + (", " + "; ".join(notes) if notes else "")
                                   + ")") if self.fused else (self.fused_note or "not attempted (COT_SHARD_IMPL=nccl)")}
        d = p.n * p.m
        self.Tl = torch.empty_like(self.sh.C)
        self.Trows = torch.empty((p.n, self.R, d), dtype=self.sh.C.dtype, device=dev)
        self.rep = torch.empty(8, dtype=torch.float64, device=dev)
        self.nf = torch.zeros(1, dtype=torch.int32, device=dev)
        self.ev = []
        self.persistent = self.fused
        self.path = (int(self.L.cot_fused_path(p.n, p.m, self.R, world, 0, self.flags)) if self.fused else 0)
        self.launches_per_step = 1 + 1 + (1 if self.fused else 3 * iters) + 3 + 1
        self.bytes_iter = float(p.n + 1) * self.R * p.m * p.C.itemsize
        q = lambda t: t.data_ptr()
        self.q = dict(C=q(self.sh.C), G=q(self.sh.G), A=q(self.sh.argmin), a=q(self.sh.alpha), b=q(self.sh.beta),
                      e=q(self.sh.eps), w=q(self.sh.w_hat), z=q(self.sh.z_hat), ws=q(self.sh.ws), Tl=q(self.Tl),
                      Tr=q(self.Trows), rep=q(self.rep), nf=q(self.nf))
        self.s = stream.cuda_stream

    def _ck(self, code, fn):
        if code != 0:
            raise RuntimeError(f"{fn} failed ({code}): {self.L.cot_last_error().decode()}")

    def step(self, record=False, C_ptr=None):
        L, q, s, sh = self.L, dict(self.q), self.s, self.sh
        if C_ptr is not None:   # e2e pipelining: this step's cost rows live in another device buffer
            q["C"] = C_ptr
        n, m, R, dt, wsn = self.n, self.m, self.R, sh.dt, sh.ws.numel()
        self._ck(L.clot_aggregate_shard(q["C"], n, R, m, dt, q["G"], q["A"], q["nf"], s), "clot_aggregate_shard")
        self._ck(L.cerot_init(q["a"], q["b"], 1, m, 1, q["z"], q["ws"], wsn, s), "cerot_init")
        if record:
            e0 = self.torch.cuda.Event(enable_timing=True)
            e1 = self.torch.cuda.Event(enable_timing=True)
            e0.record(self.stream)
        if self.fused:
            self._ck(L.cerot_iter_fused(q["a"], q["b"], q["C"], q["G"], n, m, self.row_begin, R, dt, q["e"],
                                        self.iters, 0.0, 1, self.flags, q["w"], q["z"], q["ws"], wsn, self.xchg.world,
                                        self.xchg.rank, self.xchg.xbufs, s), "cerot_iter_fused")
        else:
            self._ck(L.cerot_iter_sharded(q["a"], q["b"], q["C"], q["G"], n, m, self.row_begin, R, dt, q["e"],
                                          self.iters, 0.0, 1, self.flags, q["w"], q["z"], q["ws"], wsn,
                                          self.comm.handle, s),
                     "cerot_iter_sharded")
        if record:
            e1.record(self.stream)
            self.ev.append((e0, e1))
        self._ck(L.cerot_plan_sharded(q["a"], q["b"], q["C"], q["G"], n, m, self.row_begin, R, dt, q["e"], q["w"],
                                      q["z"], q["Tl"], q["rep"], q["ws"], wsn, self.comm.handle, s),
                 "cerot_plan_sharded")
        self._ck(L.clot_expand_shard(q["Tl"], None, n, R, m, dt, q["Tr"], s), "clot_expand_shard")

    def input_bytes(self):
        """Device bytes this rank's step reads as input (its rows of the cost blocks dominate)."""
        return self.sh.C.numel() * self.sh.C.element_size() + 2 * self.sh.alpha.numel() * 8

    def iter_kernel_ms(self):
        ts = [a.elapsed_time(b) for a, b in self.ev]
        return statistics.mean(ts), statistics.median(ts), len(ts)

    def report_row(self):
        return self.rep.cpu().numpy()

    def e2e_inputs(self):
        return self.Cl_host, self.sh.C, [(self.p.alpha, self.sh.alpha), (self.p.beta, self.sh.beta),
                                         (self.p.eps, self.sh.eps)], [self.rep, self.sh.w_hat, self.sh.z_hat]


L2_BYTES = 126e6   # B200 L2 (cudaDevAttrL2CacheSize reports 126.5 MB)


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as tdist
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    from paper_2311_13147_b200 import build as _b
    if rank == 0:
        _b.build()
    if world > 1:
        tdist.barrier()
    import paper_2311_13147_b200 as _cot
    _cot.use_current_device()   # the library's static CUDA runtime on this rank's GPU
    p, iters = make_problem(args.workload, args.iters)
    mode = "single"
    if world > 1 or os.environ.get("COT_BENCH_SHARDED") == "1":
        if p.batched:   # problem sharding (C5): a contiguous slice of the batch, no data-path collective
            from paper_2311_13147_b200 import dist as cdist
            f, cnt = cdist.problem_partition(p.B, world, rank)
            p = dataclasses.replace(p, C=p.C[f:f + cnt], alpha=p.alpha[f:f + cnt], beta=p.beta[f:f + cnt],
                                    eps=p.eps[f:f + cnt])
            mode = "problem_sharded"
        else:
            mode = "row_sharded"
    stream = torch.cuda.Stream(device=dev)

    def barrier():
        if tdist.is_initialized():
            tdist.barrier(device_ids=[local_rank])

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    with torch.cuda.stream(stream):
        R = ShardedRunner(p, iters, dev, stream, rank, world) if mode == "row_sharded" else Runner(p, iters, dev, stream)
        for _ in range(args.warmup):
            R.step()
        stream.synchronize()
        rep0 = R.report_row()
        # L2 rule: a rank whose inputs fit in twice the 126 MB L2 (C2, C3, C4 shards at N >= 2) overwrites a
        # 256 MB scratch buffer between timed steps; each step is timed by its own event pair (the flush is
        # outside them) and the step times are summed
        in_bytes = float(R.input_bytes())
        flush = in_bytes < 2 * L2_BYTES
        scratch = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        with ClockSampler(local_rank) as clk:
            barrier()
            torch.cuda.synchronize()
            for e0, e1 in evs:
                if flush:
                    scratch.fill_(1)
                e0.record(stream)
                R.step(record=True)
                e1.record(stream)
            torch.cuda.synchronize()
            barrier()
        ms_total = max_over_ranks(sum(e0.elapsed_time(e1) for e0, e1 in evs))
        l2_note = (f"per-rank inputs {in_bytes / 1e6:.1f} MB < 2 x L2 (126 MB): a 256 MB buffer is overwritten "
                   f"between timed steps (outside the per-step events)" if flush else
                   f"per-rank inputs {in_bytes / 1e6:.0f} MB > 2 x L2 (126 MB): no flush")
        ms_step = ms_total / args.steps
        it_mean, it_med, nsamp = R.iter_kernel_ms()
        it_mean = max_over_ranks(it_mean)
        # ---- e2e: the same step through the C ABI from pinned HOST buffers, copies inside the timed region
        e2e = None
        if not args.no_e2e:
            e2e = run_e2e(R, p, max(1, min(args.steps, 5)), stream)
            e2e["ms_per_step"] = max_over_ranks(e2e["ms_per_step"])
    B_total = p.B if mode != "problem_sharded" else int(os.environ.get("COT_C5_B", "4096"))
    evals_step = float(B_total) * p.n * p.m * p.m * iters
    value = evals_step / (ms_step / 1e3)
    if e2e:
        e2e["value"] = evals_step / (e2e["ms_per_step"] / 1e3)
    peak, peak_src = _peaks()
    bytes_iter = R.bytes_iter                       # this rank's C and G, streamed once per iteration
    bytes_launch = bytes_iter * iters if R.persistent else bytes_iter
    per_launch_ms = it_mean if R.persistent else it_mean / iters
    achieved = bytes_launch / (per_launch_ms / 1e3) / 1e9
    dom_share = it_mean / ms_step
    clocks = clk.summary()
    cluster = getattr(R, "path", None) in (2, 3, 4)
    if cluster:   # whole problems on chip: the bound is the SFU (one MUFU.EX2 per Gibbs evaluation), DESIGN.md §6
        ex2_launch = float(B_local_evals(p, iters)) if mode != "row_sharded" else float(p.n) * R.R * p.m * iters
        achieved_sfu = ex2_launch / (per_launch_ms / 1e3)
        mhz = clocks.get("sm_mhz") or 1965.0
        peak_sfu = 148 * 16 * mhz * 1e6
    if mode == "row_sharded":
        kernel = (("k_iter_res fused (on-chip resident shard in TMEM + shared memory, all iterations in one launch "
                   "per rank; integer column sums reduced in-kernel, exchanged through peer-mapped buffers)")
                  if R.fused and getattr(R, "path", 1) == 4 else
                  "k_iter_tma fused (persistent, all iterations in one launch per rank; column sums exchanged "
                  "in-kernel through peer-mapped LL lines)" if R.fused else
                  "per iteration: k_iter_tma rows-only + k_colsum + ncclAllReduce + k_zupdate" +
                  (f" [{R.fused_note}]" if R.fused_note else ""))
    else:
        kernel = {1: "k_iter_tma (persistent: all iterations in one launch)",
                  4: "k_iter_res (persistent, on-chip resident: the cost in TMEM + shared memory, loaded once per launch; every Gibbs term re-evaluated every iteration; integer column sums reduced in-kernel)",
                  2: "k_batch_cluster (one thread-block cluster per problem: 8 CTAs while the batch fits one wave, else 6; all iterations in one launch, on chip)",
                  3: "k_batch_chain (one thread-block cluster per problem, 8 CTAs while the batch fits one wave, else 6: one CTA runs the iteration chain, the others evaluate the n*m^2 Gibbs terms every iteration into its shared memory; all iterations in one launch, on chip)"}.get(
                      getattr(R, "path", 0), "k_rows_ldg + k_cols (one launch pair per iteration)")
    trf = _ncu_traffic_per_iter(args.workload) if world == 1 else None
    metric = _metric()
    if getattr(R, "pre", False):   # NEXT-1 is reported on its own line, never under the n*m^2 streaming metric
        metric = "C-EROT precomputed-kernel mode (Alg. 2 as written): n*m^2-equivalent evals/s (NOT the streaming metric)"
    out = {
        "metric": metric, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32" if p.C.dtype == np.float32 else "f64",
        "data": "synthetic (seeded; BASELINE.json recipe, random-rotation point clouds, no dataset)",
        "config": {"workload": p.name if mode != "problem_sharded" else f"C5_batched_B{B_total}", "B": B_total,
                   "n": p.n, "m": p.m, "d": p.d, "iters": iters,
                   "eps": float(p.eps[0]) if p.B == 1 else "per-problem 1e-2*mean(C_b)",
                   "step": "clot_aggregate + cerot_init + iters x (row pass + column pass) + cerot_plan + clot_expand",
                   "flags": hex(getattr(R, "flags", 0)) + (" (COT_DETERMINISTIC)" if getattr(R, "flags", 0) & 0x10 else ""),
                   "l2": l2_note,
                   "parallelism": {"single": "rows over the SMs of one GPU",
                                   "row_sharded": (f"rows over {world} GPUs, in-kernel exchange of the m column sums "
                                                   f"per iteration over NVLink peer memory" if getattr(R, "fused", False)
                                                   else f"rows over {world} GPUs, 1 ncclAllReduce (m fp64) per "
                                                        f"iteration"),
                                   "problem_sharded": f"problems over {world} GPUs, no collective"}[mode]},
        "roofline": ({"bound": "alu", "kernel": kernel, "achieved": achieved_sfu, "peak": peak_sfu, "unit": "ex2/s",
                      "frac": achieved_sfu / peak_sfu,
                      "peak_source": "derived: 148 SMs x 16 MUFU.EX2/clk/SM (measured 15.75-15.9, scripts/ubench) x "
                                     "the median SM clock under load (NVML)",
                      "traffic": None, "algorithmic_ex2_per_launch": ex2_launch,
                      "launch_ms_mean": per_launch_ms, "launch_samples": nsamp, "share_of_step": dom_share,
                      "us_per_iter": it_mean * 1e3 / iters} if cluster else
                     {"bound": "hbm", "kernel": kernel,
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "peak_source": peak_src,
                     "traffic": None if trf is None else trf * (iters if R.persistent else 1),
                     # the DRAM bytes ncu measured (profiles/ncu_summary.json) over the same launch time: below the
                     # algorithmic bytes where k-blocks are resident on chip (shared memory, TMEM), so this is
                     # the kernel's actual HBM utilisation, `frac` the algorithmic-bytes one
                     "traffic_frac": None if trf is None else trf * (iters if R.persistent else 1) / (per_launch_ms / 1e3) / 1e9 / peak,
                     "algorithmic_bytes_per_launch": bytes_launch, "algorithmic_bytes_per_iter": bytes_iter,
                     "launch_ms_mean": per_launch_ms, "launch_samples": nsamp, "share_of_step": dom_share,
                     "us_per_iter": it_mean * 1e3 / iters}),
        "iter_only_evals_per_s": evals_step / (it_mean / 1e3),
        "gpu_launches": R.launches_per_step * args.steps,
        "result": {"objective": float(rep0[0]), "dual": float(rep0[2]), "row_l1": float(rep0[3])},
    }
    out["exchange"] = (R.exchange if mode == "row_sharded" else
                       {"path": "none", "probe": "not needed (" + ("single GPU" if mode == "single" else
                                                                    "independent problems per rank") + ")"})
    if e2e:
        out["e2e"] = e2e
    if not args.no_cpu and rank == 0:
        out["cpu_baseline"] = cpu_baseline(p, args, args.workload)
    out["clocks"] = clocks
    if mode == "row_sharded":
        if R.xchg is not None:
            R.xchg.close()
        R.comm.close()
    return out


def B_local_evals(p, iters):
    """Gibbs evaluations (= MUFU.EX2) of one persistent launch on this rank: n*m^2 per problem per iteration."""
    return float(p.B) * p.n * p.m * p.m * iters


def run_e2e(R, p, steps, stream):
    """Host buffers -> device (pinned, async) -> step -> report + potentials back to host, every step.
    The cost copy of step k+1 runs on a second stream into the other of two device buffers while step k
    computes (independent problems stream through the device); the small inputs follow on the same copy
    stream; the results are copied back on the compute stream."""
    import torch
    hostC, devC, small, results = R.e2e_inputs()
    pin = lambda x: torch.as_tensor(np.ascontiguousarray(x)).pin_memory()
    hC = pin(hostC)
    hsmall = [(pin(h), d) for h, d in small]
    hres = [(torch.empty(r.shape, dtype=r.dtype).pin_memory(), r) for r in results]
    h2d = hC.numel() * hC.element_size() + sum(h.numel() * h.element_size() for h, _ in hsmall)
    d2h = sum(h.numel() * h.element_size() for h, _ in hres)
    bufs = [devC, torch.empty_like(devC)]
    copy_stream = torch.cuda.Stream(device=devC.device)
    big_done = [torch.cuda.Event() for _ in bufs]
    big_free = [torch.cuda.Event() for _ in bufs]
    small_done, small_free = torch.cuda.Event(), torch.cuda.Event()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)

    # All host->device copies go through the copy stream in issue order (one DMA queue): the cost of step k+1
    # (double-buffered) is issued before step k computes, the small inputs of step k+1 right after step k
    # released them; the step waits only for its own copies.
    def issue_big(k):
        b = k % len(bufs)
        if k >= len(bufs):
            copy_stream.wait_event(big_free[b])
        else:
            copy_stream.wait_stream(stream)
        with torch.cuda.stream(copy_stream):
            bufs[b].copy_(hC, non_blocking=True)
        big_done[b].record(copy_stream)

    def issue_small(k):
        if k > 0:
            copy_stream.wait_event(small_free)
        with torch.cuda.stream(copy_stream):
            for h, d in hsmall:
                d.copy_(h, non_blocking=True)
        small_done.record(copy_stream)

    issue_big(0)
    issue_small(0)
    for k in range(steps):
        b = k % len(bufs)
        if k + 1 < steps:
            issue_big(k + 1)
        stream.wait_event(big_done[b])
        stream.wait_event(small_done)
        R.step(C_ptr=bufs[b].data_ptr())
        big_free[b].record(stream)
        small_free.record(stream)
        for h, d in hres:
            h.copy_(d, non_blocking=True)
        if k + 1 < steps:
            issue_small(k + 1)
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    return {"value": None, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": ms, "steps": steps,
            "pipelining": "H2D of step k+1's cost (second stream, double-buffered) overlaps step k",
            "api": "C ABI (clot_aggregate, cerot_init/iter/plan, clot_expand; sharded variants for N>1)"}


# ------------------------------------------------------------------------------------------ oracle arm
# The oracle as it stands (fp64 NumPy, never tuned for this), on the box's host cores: one BLAS
# thread per worker process, one worker per core of sched_getaffinity, each worker running the oracle on its own
# problem of the workload (C5: problem `worker` of the batch; C2: the eps sweep's problems round-robin; C3/C4: the
# single problem, i.e. independent replicas). Workers are spawned (no fork of a CUDA process) and build their
# problem from the seeded generators before the timed region.
_W = {}


def _worker_problem(workload: str, w: int):
    import synthetic
    if workload == "C4":
        return synthetic.c4_large()
    if workload == "C3":
        return synthetic.c3_image()
    if workload == "C2":
        return synthetic.c2_sweep().single(w % 3)
    if workload == "C2e2":
        return synthetic.c2_ring(eps_factor=1e-2)
    if workload == "C5":
        return synthetic.c5_batched(B=1, first=w % 4096).single(0)
    raise SystemExit(f"unknown workload {workload}")


def _worker_init(workload: str, counter, lock):
    try:
        from threadpoolctl import threadpool_limits
        _W["lim"] = threadpool_limits(1)
    except Exception:
        pass
    with lock:
        w = counter.value
        counter.value += 1
    _W["q"] = _worker_problem(workload, w)
    _W["w"] = w


def _worker_run(args):
    """k iterations of the oracle's cyclic Sinkhorn in `form` on this worker's problem, after a barrier (so the
    all-core runs overlap). Returns (evaluations-equivalent n*m^2*k, seconds)."""
    import oracle
    k, form, barrier = args
    q = _W["q"]
    if barrier is not None:
        barrier.wait()
    t = time.perf_counter()
    oracle.cyclic_sinkhorn(q.alpha, q.beta, q.C, float(q.eps[0]), k, form=form)
    return float(q.n * q.m * q.m * k), time.perf_counter() - t


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


class OraclePool:
    """All host cores running the oracle (one single-threaded worker per core)."""

    def __init__(self, workload: str, cores: int | None = None):
        import multiprocessing as mp
        self.ctx = mp.get_context("spawn")
        self.cores = cores or len(os.sched_getaffinity(0))
        self.mgr = self.ctx.Manager()
        counter, lock = self.mgr.Value("i", 0), self.mgr.Lock()
        self.pool = self.ctx.Pool(self.cores, initializer=_worker_init, initargs=(workload, counter, lock))
        self.pool.map(_worker_run, [(0, "stream", None)] * self.cores, chunksize=1)   # all workers built

    def run(self, k: int, form: str, workers: int | None = None):
        """k iterations on `workers` workers at once; returns (total evals, wall seconds, per-worker seconds)."""
        P = workers or self.cores
        bar = self.mgr.Barrier(P) if P > 1 else None
        t = time.perf_counter()
        res = self.pool.map(_worker_run, [(k, form, bar)] * P, chunksize=1)
        wall = time.perf_counter() - t
        ev = sum(r[0] for r in res)
        return ev, max(r[1] for r in res), wall

    def close(self):
        self.pool.close()
        self.pool.join()
        self.mgr.shutdown()


def _iters_for(p, seconds: float, rate: float = 4.0e7) -> int:
    q = p.single(0) if p.batched else p
    return max(1, min(500, int(seconds * rate / (q.n * q.m * q.m))))


def cpu_baseline(p, args, workload: str):
    """The oracle as it stands timed on this box's host cores on a bounded sample of the same workload: the
    streaming form (the same n*m^2 work per iteration as the kernel) on one core and on all cores, and Alg. 2 with
    K precomputed (the paper's own CPU algorithm; its rate counted in n*m^2-equivalent evaluations, the one-off
    log K build inside the timed region) on all cores. ~25 s in total."""
    sec = float(os.environ.get("COT_CPU_BASELINE_SECONDS", "6"))   # per leg (tests use less)
    pool = OraclePool(workload)
    try:
        k = _iters_for(p, sec)
        ev1, t1, _ = pool.run(k, "stream", workers=1)
        evP, tP, _ = pool.run(k, "stream")
        kk = max(k, _iters_for(p, sec, rate=4.0e7 * p.n))
        evK, tK, _ = pool.run(kk, "kernel")
    finally:
        pool.close()
    q = p.single(0) if p.batched else p
    return {"value": evP / tP, "unit": UNIT, "cores": pool.cores, "kind": "oracle",
            "per_core": ev1 / t1, "all_core": evP / tP,
            "kernel_form": {"value": evK / tK, "unit": "n*m^2-equivalent evals/s (Alg. 2, K precomputed once)",
                            "iters": kk, "cores": pool.cores, "seconds": tK},
            "cpu_model": _cpu_model(),
            "sample": (f"{workload}: {k} cyclic Sinkhorn iterations per worker (oracle streaming form, fp64 NumPy, "
                       f"1 BLAS thread), 1 worker ({t1:.1f} s) and {pool.cores} workers at once ({tP:.1f} s); "
                       f"kernel form {kk} iterations x {pool.cores} workers ({tK:.1f} s); "
                       f"each worker its own problem ({q.name} recipe)")}


def run_reference(args):
    """--impl reference: the oracle timed on the host's cores. One step = one cyclic Sinkhorn
    iteration (streaming form: the same n*m^2 work as the kernel) on every core at once, each worker on its own
    problem of the workload -- a bounded sample of the full solve; value = evaluations / step time."""
    p, iters = make_problem(args.workload, args.iters)
    pool = OraclePool(args.workload)
    try:
        for _ in range(args.warmup):
            pool.run(1, "stream")
        tot_ev, tot_t = 0.0, 0.0
        for _ in range(args.steps):
            ev, t, wall = pool.run(1, "stream")
            tot_ev += ev
            tot_t += wall
    finally:
        pool.close()
    ms = tot_t / args.steps * 1e3
    value = tot_ev / tot_t
    q = p.single(0) if p.batched else p
    sample = (f"{args.steps} steps x 1 iteration (oracle streaming form, fp64 NumPy, 1 BLAS thread per worker) on "
              f"{pool.cores} worker processes at once, each on its own problem of the {args.workload} recipe")
    return {"impl": "reference", "metric": _metric(), "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded; BASELINE.json recipe)",
            "config": {"workload": p.name, "B": p.B, "n": q.n, "m": q.m, "d": q.d, "iters_per_step": 1,
                       "full_solve_iters": iters, "sample": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": pool.cores, "kind": "oracle", "sample": sample,
                             "cpu_model": _cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    # stdout carries exactly one JSON line: everything else written to fd 1 by native code (e.g. NCCL's version
    # banner at its first collective) goes to stderr; the JSON line is written to the saved stdout
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    global _JSON_OUT
    _JSON_OUT = os.fdopen(json_fd, "w")
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--iters", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        # one process per GPU: N > 1 must be launched by torchrun (WORLD_SIZE = N); never report n_gpus silently
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch N > 1 with "
              f"`python -m torch.distributed.run --nproc-per-node {args.gpus} ... bench.py --gpus {args.gpus}`",
              file=sys.stderr)
        return 2
    if args.impl == "reference":
        if rank != 0:
            return 0
        print(json.dumps(run_reference(args)), file=_JSON_OUT, flush=True)
        return 0
    force_sharded = os.environ.get("COT_BENCH_SHARDED") == "1"   # exercise the row-sharded path at N = 1
    if world > 1 or force_sharded:
        import torch
        torch.cuda.set_device(local_rank)
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    out = run_ours(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(out), file=_JSON_OUT, flush=True)
    if torch_dist_initialized():
        import torch.distributed as tdist
        tdist.destroy_process_group()
    return 0


def torch_dist_initialized() -> bool:
    try:
        import torch.distributed as tdist
        return tdist.is_available() and tdist.is_initialized()
    except Exception:
        return False


if __name__ == "__main__":
    sys.exit(main())
