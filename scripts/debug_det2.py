import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2311_13147_b200 as cot
import synthetic
dev = torch.device("cuda:0")
p = synthetic.c4_large(m=512, n=16)
D = lambda x: torch.as_tensor(np.ascontiguousarray(x), device=dev)
def run(splits):
    pr = cot.CerotProblem(D(p.C), D(p.alpha), D(p.beta), D(p.eps)).init()
    for k in splits: pr.iterate(k, flags=cot.COT_DETERMINISTIC)
    torch.cuda.synchronize()
    return pr.w_hat.cpu().numpy(), pr.z_hat.cpu().numpy()
a = run([1, 1]); b = run([1, 1]); c = run([2])
print("1+1 vs 1+1: w", int((a[0] != b[0]).sum()), "z", int((a[1] != b[1]).sum()))
i = np.nonzero(a[1] != c[1])[0]
print("1+1 vs 2: z idx", i[:8], "rel diff", (np.abs(a[1][i] - c[1][i]) / np.abs(c[1][i]))[:8])
