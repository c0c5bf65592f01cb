"""NEXT-4 timing: the host network simplex (clot_small_lot) against HiGHS (the oracle's LP) on the small LOT
of C-LOT instances: App. D sizes (m = 100, 200 at n = 50: Table 1's d = 5000, 10000), C5 (m = 128)
and C3/C4 sizes (m = 1024). Prints one JSON line per instance (host seconds, values, pivots)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synthetic  # noqa: E402
from paper_2311_13147_b200 import host_lp  # noqa: E402


def run(name, alpha, beta, G, highs=True):
    t0 = time.perf_counter()
    v, S, u, w, piv = host_lp.small_lot(alpha, beta, G, duals=True)
    t1 = time.perf_counter()
    out = {"instance": name, "m": G.shape[0], "netsimplex_s": t1 - t0, "pivots": piv, "value": v,
           "nnz": int((S > 0).sum())}
    if highs:
        t2 = time.perf_counter()
        ref, _ = oracle.lot(alpha, beta, G)
        out.update(highs_s=time.perf_counter() - t2, highs_value=ref, rel_diff=abs(v - ref) / max(abs(ref), 1e-300))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for d in (5000, 10000):
        p = synthetic.appd_synthetic(0, d=d)
        G, _ = oracle.aggregate(p.C)
        run(f"appD_d{d}_n{p.n}", p.alpha, p.beta, G)
    q = synthetic.c5_batched(B=1)
    G, _ = oracle.aggregate(q.C[0])
    run("C5_problem0", q.alpha[0], q.beta[0], G.astype(np.float64))
    r = synthetic.c4_large()
    G, _ = oracle.aggregate(r.C)
    run("C4_m1024", r.alpha, r.beta, G.astype(np.float64), highs="--highs-1024" in sys.argv)
