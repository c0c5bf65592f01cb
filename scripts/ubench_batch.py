"""Cluster-resident batched kernel on a C5 slice (B problems, ITERS iterations): time per iteration-wave."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_13147_b200 as cot
import synthetic
B = int(os.environ.get("B", "144")); iters = int(os.environ.get("ITERS", "50"))
p = synthetic.c5_batched(B=B)
dev = torch.device("cuda:0")
prob = cot.CerotProblem(torch.as_tensor(p.C, device=dev), torch.as_tensor(p.alpha, device=dev),
                        torch.as_tensor(p.beta, device=dev), torch.as_tensor(p.eps, device=dev))
for rep in range(2):
    prob.init()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); prob.iterate(iters); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
waves = -(-B // 18)
print(f"B={B} iters={iters}: {ms:.3f} ms, {ms*1e3/iters/waves:.2f} us per iteration per cluster wave, "
      f"{B*16*128*128*iters/ms/1e9:.3e} evals/s")
