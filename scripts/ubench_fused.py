"""Protocol overhead of the fused multi-GPU exchange, measured on ONE GPU: C4 (or --m/--n) as V emulated ranks
in one cooperative launch (each virtual rank on 1/V of the SMs, in-kernel LL-line exchange every iteration)
against the unsharded persistent kernel on all SMs. Same total work and SMs, so the difference is the cost
of the exchange protocol (not a multi-GPU scaling number). Prints one JSON line per V."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthetic  # noqa: E402
import paper_2311_13147_b200 as cot  # noqa: E402
from paper_2311_13147_b200 import dist as cdist  # noqa: E402


def timed(fn, reps=3):
    ts = []
    for _ in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts[1:])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=1024)
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--flags", type=lambda x: int(x, 0), default=0, help="diagnostic flags (COT_DIAG_*)")
    ap.add_argument("--shard-alone", type=int, default=0,
                    help="G > 0: run rank 0's shard of a G-way row partition ALONE on this GPU (cerot_iter_fused, "
                         "nranks = 1, exchange with itself): the per-GPU work and local sync of a G-GPU run, "
                         "without the NVLink latency")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    p = synthetic.c4_large(m=a.m, n=a.n)
    D = lambda x: torch.as_tensor(np.ascontiguousarray(x), device=dev)
    if a.shard_alone:
        G = a.shard_alone
        b0, R = cdist.row_partition(p.m, G, 0)
        sh = cdist.ShardedCerot(D(p.C[:, b0:b0 + R, :]), D(p.alpha), D(p.beta), float(p.eps[0]), b0, p.m)
        x = cdist.PeerExchange(p.m)
        ms = timed(lambda: sh.init().iterate_fused(x, a.iters, flags=a.flags))
        print(json.dumps({"mode": f"shard_alone_1_of_{G}", "rows": R, "m": a.m, "n": a.n, "flags": a.flags,
                          "us_per_iter": ms * 1e3 / a.iters}))
        x.close()
        return
    prob = cot.CerotProblem(D(p.C), D(p.alpha), D(p.beta), p.eps)
    ms = timed(lambda: prob.init().iterate(a.iters))
    print(json.dumps({"mode": "unsharded", "m": a.m, "n": a.n, "us_per_iter": ms * 1e3 / a.iters}))
    for V in [int(v) for v in a.ranks.split(",")]:
        shards = []
        for r in range(V):
            b0, R = cdist.row_partition(p.m, V, r)
            shards.append(cdist.ShardedCerot(D(p.C[:, b0:b0 + R, :]), D(p.alpha), D(p.beta), float(p.eps[0]), b0, p.m))
        xb = cdist.emulate_fused([s.init() for s in shards], 1)

        def run():
            for s in shards:
                s.init()
            cdist.emulate_fused(shards, a.iters, xbufs=xb)
        ms = timed(run)
        print(json.dumps({"mode": f"fused_emulated_{V}_ranks", "m": a.m, "n": a.n, "us_per_iter": ms * 1e3 / a.iters}))
        cdist.free_xbufs(xb)


if __name__ == "__main__":
    main()
