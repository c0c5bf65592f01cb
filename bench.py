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
    elif workload == "C2":
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
        self.flags = int(os.environ.get("COT_BENCH_FLAGS", "0"))
        # the persistent TMA kernel runs all iterations in one launch (B == 1, fp32, m % 4 == 0)
        self.persistent = (self.B == 1 and self.dt == cot.COT_F32 and self.m % 4 == 0 and not (self.flags & 2))
        self.launches_per_step = 1 + 1 + (1 if self.persistent else 2 * iters) + 2 + 1

    def _ck(self, code, fn):
        if code != 0:
            raise RuntimeError(f"{fn} failed ({code}): {self.L.cot_last_error().decode()}")

    def step(self, record=False):
        L, q, s = self.L, self.ptr, self.s
        B, n, m, dt = self.B, self.n, self.m, self.dt
        wsn = self.ws.numel()
        self._ck(L.clot_aggregate(q["C"], B, n, m, dt, q["G"], q["A"], None, s), "clot_aggregate")
        self._ck(L.cerot_init(q["a"], q["b"], B, m, 1, q["z"], q["ws"], wsn, s), "cerot_init")
        if record:
            e0 = self.torch.cuda.Event(enable_timing=True)
            e1 = self.torch.cuda.Event(enable_timing=True)
            e0.record(self.stream)
        self._ck(L.cerot_iter(q["a"], q["b"], q["C"], q["G"], B, n, m, dt, q["e"], self.iters, 0.0, 1, self.flags,
                              q["w"], q["z"], q["ws"], wsn, s), "cerot_iter")
        if record:
            e1.record(self.stream)
            self.ev.append((e0, e1))
        self._ck(L.cerot_plan(q["a"], q["b"], q["C"], q["G"], B, n, m, dt, q["e"], q["w"], q["z"], q["Tb"], q["rep"],
                              q["ws"], wsn, s), "cerot_plan")
        self._ck(L.clot_expand(q["Tb"], None, B, n, m, dt, q["Tf"], s), "clot_expand")

    def iter_kernel_ms(self):
        """Device time of the iteration launch(es) of each timed step (CUDA events on our stream)."""
        ts = [a.elapsed_time(b) for a, b in self.ev]
        return statistics.mean(ts), statistics.median(ts), len(ts)


def run_ours(args, rank, world, local_rank):
    import torch
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    from paper_2311_13147_b200 import build as _b
    if rank == 0:
        _b.build()
    if world > 1:
        torch.distributed.barrier()
    p, iters = make_problem(args.workload, args.iters)
    if world > 1:
        raise SystemExit("multi-GPU row sharding: see bench_sharded (not in this build)")
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        R = Runner(p, iters, dev, stream)
        for _ in range(args.warmup):
            R.step()
        stream.synchronize()
        rep0 = R.rep.cpu().numpy()[0]
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        with ClockSampler(local_rank) as clk:
            torch.cuda.synchronize()
            start.record(stream)
            for _ in range(args.steps):
                R.step(record=True)
            end.record(stream)
            torch.cuda.synchronize()
        ms_total = start.elapsed_time(end)
        ms_step = ms_total / args.steps
        it_mean, it_med, nsamp = R.iter_kernel_ms()
        # ---- e2e: the same step through the C ABI from pinned HOST buffers, copies inside the timed region
        e2e = run_e2e(R, p, max(1, min(args.steps, 3)), stream) if not args.no_e2e else None
    evals_step = float(p.B) * p.n * p.m * p.m * iters
    value = evals_step / (ms_step / 1e3)
    peak, peak_src = _peaks()
    bytes_iter = float(p.B) * (p.n + 1) * p.m * p.m * p.C.itemsize     # C and G streamed once per iteration
    bytes_launch = bytes_iter * iters if R.persistent else bytes_iter
    per_launch_ms = it_mean if R.persistent else it_mean / iters
    achieved = bytes_launch / (per_launch_ms / 1e3) / 1e9
    dom_share = it_mean / ms_step
    out = {
        "metric": _metric(), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32" if p.C.dtype == np.float32 else "f64",
        "data": "synthetic (seeded; BASELINE.json recipe, random-rotation point clouds, no dataset)",
        "config": {"workload": p.name, "B": p.B, "n": p.n, "m": p.m, "d": p.d, "iters": iters,
                   "eps": float(p.eps[0]) if p.B == 1 else "per-problem 1e-2*mean(C_b)",
                   "step": "clot_aggregate + cerot_init + iters x (cerot_rows + cerot_cols) + cerot_plan + clot_expand",
                   "l2": f"inputs ({p.C.nbytes / 1e6:.0f} MB of cost) larger than L2 (126 MB): no flush",
                   "parallelism": f"rows/units over {torch.cuda.get_device_properties(dev).multi_processor_count} SMs"},
        "roofline": {"bound": "hbm",
                     "kernel": ("k_iter_tma (persistent: all iterations in one launch)" if R.persistent
                                else "k_rows_ldg + k_cols (one launch pair per iteration)"),
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "peak_source": peak_src,
                     "traffic": (None if _ncu_traffic_per_iter(args.workload) is None else
                                 _ncu_traffic_per_iter(args.workload) * (iters if R.persistent else 1)),
                     "algorithmic_bytes_per_launch": bytes_launch, "algorithmic_bytes_per_iter": bytes_iter,
                     "launch_ms_mean": per_launch_ms, "launch_samples": nsamp, "share_of_step": dom_share,
                     "us_per_iter": it_mean * 1e3 / iters},
        "iter_only_evals_per_s": float(p.B) * p.n * p.m * p.m * iters / (it_mean / 1e3),
        "gpu_launches": R.launches_per_step * args.steps,
        "result": {"objective": float(rep0[0]), "dual": float(rep0[2]), "row_l1": float(rep0[3])},
    }
    if e2e:
        out["e2e"] = e2e
    if not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(p, args)
    out["clocks"] = clk.summary()
    return out


def run_e2e(R, p, steps, stream):
    """Host buffers -> device (pinned, async) -> step -> report + potentials back to host, per step."""
    import torch
    pin = lambda x: torch.as_tensor(np.ascontiguousarray(x)).pin_memory()
    hC, ha, hb, he = pin(p.C), pin(p.alpha), pin(p.beta), pin(p.eps)
    hrep = torch.empty((R.B, 8), dtype=torch.float64).pin_memory()
    hw = torch.empty_like(R.w, device="cpu").pin_memory()
    hz = torch.empty_like(R.z, device="cpu").pin_memory()
    h2d = hC.numel() * hC.element_size() + (ha.numel() + hb.numel() + he.numel()) * 8
    d2h = (hrep.numel() + hw.numel() + hz.numel()) * 8
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        R.C.copy_(hC, non_blocking=True)
        R.alpha.copy_(ha, non_blocking=True)
        R.beta.copy_(hb, non_blocking=True)
        R.eps.copy_(he, non_blocking=True)
        R.step()
        hrep.copy_(R.rep, non_blocking=True)
        hw.copy_(R.w, non_blocking=True)
        hz.copy_(R.z, non_blocking=True)
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    evals = float(p.B) * p.n * p.m * p.m * R.iters
    return {"value": evals / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": ms, "steps": steps, "api": "C ABI (clot_aggregate, cerot_init/rows/cols/plan, clot_expand)"}


# ------------------------------------------------------------------------------------------ oracle arm
def _oracle_iters(p, iters):
    import oracle
    q = p.single(0) if p.batched else p
    t = time.perf_counter()
    oracle.cyclic_sinkhorn(q.alpha, q.beta, q.C, float(q.eps[0]), iters, form="stream")
    return time.perf_counter() - t, q


def cpu_baseline(p, args):
    """The oracle as it stands (fp64 NumPy, streaming form = the same n*m^2 work per iteration), timed on
    the host on a bounded sample: a few iterations of one problem of the same workload."""
    try:
        from threadpoolctl import threadpool_limits
        lim = threadpool_limits(1)
    except Exception:
        lim = None
    q = p.single(0) if p.batched else p
    per_iter = q.n * q.m * q.m
    k = max(1, min(50, int(12.0 / max(per_iter / 4.0e7, 1e-6))))     # ~10-20 s at ~40M evals/s
    dt, _ = _oracle_iters(p, k)
    if lim is not None:
        lim.unregister() if hasattr(lim, "unregister") else None
    return {"value": per_iter * k / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{q.name}: {k} cyclic Sinkhorn iterations (oracle streaming form, fp64 NumPy, 1 thread), "
                      f"{dt:.1f} s", "host_cores_available": len(os.sched_getaffinity(0))}


def run_reference(args):
    """--impl reference: the oracle timed on the host; one step = one cyclic Sinkhorn
    iteration (streaming form) of the same workload, a bounded sample of the full solve."""
    p, iters = make_problem(args.workload, args.iters)
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    for _ in range(args.warmup):
        _oracle_iters(p, 1)
    t = time.perf_counter()
    for _ in range(args.steps):
        dt, q = _oracle_iters(p, 1)
    total = time.perf_counter() - t
    ms = total / args.steps * 1e3
    q = p.single(0) if p.batched else p
    value = q.n * q.m * q.m / (ms / 1e3)
    return {"impl": "reference", "metric": _metric(), "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded; BASELINE.json recipe)",
            "config": {"workload": q.name, "n": q.n, "m": q.m, "d": q.d, "iters_per_step": 1,
                       "full_solve_iters": iters},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{args.steps} steps x 1 iteration of {q.name} (oracle streaming form, fp64)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
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
    if args.impl == "reference":
        if rank != 0:
            return 0
        print(json.dumps(run_reference(args)), flush=True)
        return 0
    if world > 1:
        import torch
        torch.distributed.init_process_group("nccl")
    out = run_ours(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(out), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
