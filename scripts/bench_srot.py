"""NEXT-3 measurement: C-SROT with the squared regulariser (alternating maximisation) on the device --
device time per sweep (one w-step + one z-step, each solving every coordinate by safeguarded Newton, every
Newton step a streamed pass over the coordinate's n*m costs) on the C2 and C3 shapes, fixed sweep counts."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthetic  # noqa: E402
import paper_2311_13147_b200 as cot  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    D = lambda x: torch.as_tensor(np.ascontiguousarray(x), device=dev)
    for name, p, gam, sweeps in (("C2_ring", synthetic.c2_ring(), 1.0, 50), ("C3_image", synthetic.c3_image(), 1.0, 50)):
        C, a, b = D(p.C), D(p.alpha), D(p.beta)
        cot.csrot_solve(C, a, b, gam, max_sweeps=2)   # warm-up
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        _, _, _, rep = cot.csrot_solve(C, a, b, gam, max_sweeps=sweeps)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(json.dumps({"workload": name, "n": p.n, "m": p.m, "gamma": gam, "sweeps": sweeps, "ms": ms,
                          "us_per_sweep": ms * 1e3 / sweeps,
                          "cost_visits_per_s_lower_bound": 2.0 * p.n * p.m * p.m * sweeps / (ms / 1e3),
                          "objective": rep[0]["objective"], "col_l1": rep[0]["col_l1"]}), flush=True)


if __name__ == "__main__":
    main()
