"""cerot_solve to tolerance ("until convergence", decided on the device): wall time of the whole solve
(aggregate, init, iterations, plan, report; one host synchronisation) and us per iteration, for C1 (fp64: the
generic kernels as one CUDA graph with a device-side while loop) and C3 (one persistent launch). JSON lines."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthetic  # noqa: E402
import paper_2311_13147_b200 as cot  # noqa: E402

dev = torch.device("cuda:0")
D = lambda x: torch.as_tensor(np.ascontiguousarray(x), device=dev)  # noqa: E731
for name, p, ce in (("C1", synthetic.c1_tiny(), 1), ("C3", synthetic.c3_image(pair=1), 10)):
    C, a, b = D(p.C), D(p.alpha), D(p.beta)
    tol = p.tol if p.tol > 0 else 1e-9
    best, reps = 1e9, None
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, _, _, reps = cot.cerot_solve(C, a, b, p.eps, tol=tol, max_iter=100000, check_every=ce)
        best = min(best, time.perf_counter() - t0)
    it = reps[0]["iters"]
    print(json.dumps({"workload": name, "tol": tol, "check_every": ce, "iters": it, "converged": reps[0]["converged"],
                      "solve_ms": best * 1e3, "us_per_iter_incl_setup": best * 1e6 / it,
                      "path": int(cot.lib().cot_iter_path(p.B, p.n, p.m, 1 if p.C.dtype == np.float64 else 0, 0)),
                      "host_syncs": 1, "objective": reps[0]["objective"]}), flush=True)
