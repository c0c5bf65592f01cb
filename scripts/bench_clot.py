"""C-LOT end to end (Alg. 1) on the paper's own synthetic workload (App. D: d = 5000,
10000 at n = 50, lambda irrelevant for LOT) and on a C5 problem: host cost blocks -> device (H2D),
clot_aggregate on the GPU, the small LOT by the host network simplex (NEXT-4), the lift + dense d x d
expansion on the GPU, the plan's checksum back to the host. Wall time per instance (the paper's timed
interval "between inputting the data and outputting the optimal solution"), next to the paper's
cyclic network simplex times (Table 1, i7-10750H laptop, Python + LEMON: context only)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthetic  # noqa: E402
import paper_2311_13147_b200 as cot  # noqa: E402
from paper_2311_13147_b200 import host_lp  # noqa: E402

PAPER = {5000: 0.056, 10000: 0.329}   # Table 1, cyclic network simplex at n = 50, seconds


def one(C_host, alpha, beta, dev):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    C = torch.as_tensor(C_host).to(dev, non_blocking=False)
    G, A = cot.clot_aggregate(C)
    Gh = G.double().cpu().numpy()
    t1 = time.perf_counter()
    val, S = host_lp.small_lot(alpha, beta, Gh)
    t2 = time.perf_counter()
    T = cot.clot_expand(torch.as_tensor(S, dtype=C.dtype, device=dev), C.shape[0], argmin=A)
    chk = float(T.sum().item())
    t3 = time.perf_counter()
    return C.shape[0] * val, chk, t1 - t0, t2 - t1, t3 - t2, t3 - t0


def main():
    dev = torch.device("cuda:0")
    for d in (5000, 10000):
        ts = []
        for seed in range(5):
            p = synthetic.appd_synthetic(seed, d=d)
            C = np.ascontiguousarray(p.C.astype(np.float64))
            one(C, p.alpha, p.beta, dev) if seed == 0 else None   # warm-up (module load, allocator)
            val, chk, ta, tl, te, tt = one(C, p.alpha, p.beta, dev)
            ts.append(tt)
            print(json.dumps({"workload": f"appD_d{d}_n{p.n}_seed{seed}", "value_full": val, "plan_mass": chk,
                              "s_h2d_aggregate": ta, "s_host_lp": tl, "s_expand_d2h": te, "s_total": tt}), flush=True)
        print(json.dumps({"workload": f"appD_d{d}_n50", "mean_s": float(np.mean(ts)),
                          "paper_cyclic_network_simplex_s": PAPER[d],
                          "note": "paper: i7-10750H laptop, Python + LEMON (context only)"}), flush=True)
    q = synthetic.c5_batched(B=1)
    one(q.C[0], q.alpha[0], q.beta[0], dev)
    val, chk, ta, tl, te, tt = one(q.C[0], q.alpha[0], q.beta[0], dev)
    print(json.dumps({"workload": "C5_problem0_d2048_n16", "value_full": val, "s_h2d_aggregate": ta, "s_host_lp": tl,
                      "s_expand_d2h": te, "s_total": tt}), flush=True)


if __name__ == "__main__":
    main()
