"""Cluster-resident kernel: time of ITERS iterations for B problems, B around the number of co-resident
8-CTA clusters (wave structure of the C5 batch)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_13147_b200 as cot
import synthetic
iters = int(os.environ.get("ITERS", "200"))
dev = torch.device("cuda:0")
full = synthetic.c5_batched(B=64)
for B in [1, 8, 14, 15, 16, 17, 18, 19, 32, 36, 64]:
    C = torch.as_tensor(full.C[:B], device=dev)
    prob = cot.CerotProblem(C, torch.as_tensor(full.alpha[:B], device=dev), torch.as_tensor(full.beta[:B], device=dev),
                            torch.as_tensor(full.eps[:B], device=dev))
    best = 1e9
    for rep in range(3):
        prob.init()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); prob.iterate(iters); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"B={B:3d}: {best*1e3/iters:.3f} us per iteration", flush=True)
