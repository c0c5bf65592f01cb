"""C2 (one ring problem, m = 128, n = 8) through the cluster-resident kernel: us per iteration (500 iterations)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_13147_b200 as cot
import synthetic
dev = torch.device("cuda:0")
p = synthetic.c2_ring(eps_factor=float(os.environ.get("EPSF", "1e-2")))
prob = cot.CerotProblem(torch.as_tensor(p.C, device=dev), torch.as_tensor(p.alpha, device=dev),
                        torch.as_tensor(p.beta, device=dev), p.eps)
best = 1e9
for rep in range(3):
    prob.init()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); prob.iterate(500); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(f"C2 shape {os.environ.get('COT_BATCH_SHAPE', 'default')}: {best * 1e3 / 500:.3f} us per iteration")
