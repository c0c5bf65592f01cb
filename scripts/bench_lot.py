"""NEXT-4 timing: the host network simplex (clot_small_lot) against SciPy's HiGHS LP on the small LOT of C-LOT
instances: App. D sizes (m = 100, 200 at n = 50: Table 1's d = 5000, 10000), C5 (m = 128) and C3/C4
sizes (m = 1024). The HiGHS LP is set up here (timing tooling: it does not use oracle/, which only tests,
smoke() and bench.py's CPU legs may run). Prints one JSON line per instance (host seconds, values, pivots)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scipy.optimize  # noqa: E402
import scipy.sparse  # noqa: E402

import synthetic  # noqa: E402
from paper_2311_13147_b200 import host_lp  # noqa: E402


def highs_value(a, b, G):
    """min <G, S> s.t. S 1 = a, S^T 1 = b, S >= 0 with SciPy's HiGHS (the comparison solver)."""
    p, q = G.shape
    A_eq = scipy.sparse.vstack([scipy.sparse.kron(scipy.sparse.eye(p), np.ones((1, q))),
                                scipy.sparse.kron(np.ones((1, p)), scipy.sparse.eye(q))]).tocsr()
    res = scipy.optimize.linprog(G.ravel(), A_eq=A_eq, b_eq=np.concatenate([a, b]), bounds=(0, None),
                                 method="highs", options={"primal_feasibility_tolerance": 1e-10,
                                                          "dual_feasibility_tolerance": 1e-10})
    if res.status != 0:
        raise RuntimeError(f"LP failed: {res.message}")
    return float(G.ravel() @ res.x)


def aggregate(C):
    """G = min_k C_k (the LP's cost; its values are all the timing needs), fp64."""
    return np.asarray(C).min(axis=0).astype(np.float64)


def run(name, alpha, beta, G, highs=True):
    t0 = time.perf_counter()
    v, S, u, w, piv = host_lp.small_lot(alpha, beta, G, duals=True)
    t1 = time.perf_counter()
    out = {"instance": name, "m": G.shape[0], "netsimplex_s": t1 - t0, "pivots": piv, "value": v,
           "nnz": int((S > 0).sum())}
    if highs:
        t2 = time.perf_counter()
        ref = highs_value(np.asarray(alpha, np.float64), np.asarray(beta, np.float64), G)
        out.update(highs_s=time.perf_counter() - t2, highs_value=ref, rel_diff=abs(v - ref) / max(abs(ref), 1e-300))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for d in (5000, 10000):
        p = synthetic.appd_synthetic(0, d=d)
        run(f"appD_d{d}_n{p.n}", p.alpha, p.beta, aggregate(p.C))
    q = synthetic.c5_batched(B=1)
    run("C5_problem0", q.alpha[0], q.beta[0], aggregate(q.C[0]))
    r = synthetic.c4_large()
    run("C4_m1024", r.alpha, r.beta, aggregate(r.C), highs="--highs-1024" in sys.argv)
