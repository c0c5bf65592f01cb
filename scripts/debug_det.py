"""Deterministic mode: which factor changes bits (launch split / CTA count / ranks)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2311_13147_b200 as cot
import synthetic
dev = torch.device("cuda:0")
p = synthetic.c4_large(m=512, n=16)
D = lambda x: torch.as_tensor(np.ascontiguousarray(x), device=dev)
def run(splits, ctas=None):
    if ctas: os.environ["COT_MAX_CTAS"] = str(ctas)
    else: os.environ.pop("COT_MAX_CTAS", None)
    pr = cot.CerotProblem(D(p.C), D(p.alpha), D(p.beta), D(p.eps)).init()
    for k in splits: pr.iterate(k, flags=cot.COT_DETERMINISTIC)
    torch.cuda.synchronize()
    return pr.w_hat.cpu().numpy().view(np.uint64), pr.z_hat.cpu().numpy().view(np.uint64)
a = run([25]); b = run([10, 15]); c = run([25], 100); d = run([1]*25); e = run([25])
for name, x in (("split10+15", b), ("ctas100", c), ("split1x25", d), ("repeat", e)):
    print(name, "w diff", int((x[0] != a[0]).sum()), "z diff", int((x[1] != a[1]).sum()))
for k in (1, 2, 3):
    a1 = run([k]); b1 = run([k], 100)
    print("iters", k, "ctas100 w diff", int((a1[0] != b1[0]).sum()), "z diff", int((a1[1] != b1[1]).sum()))
a = run([2]); b = run([1, 1])
wi = np.nonzero(a[0] != b[0])[0]; zi = np.nonzero(a[1] != b[1])[0]
print("2 vs 1+1: w diff rows", wi[:20], "(mod 4:", np.bincount(wi % 4, minlength=4), ") z diff", zi[:20])
a = run([3]); b = run([2, 1])
wi = np.nonzero(a[0] != b[0])[0]; zi = np.nonzero(a[1] != b[1])[0]
print("3 vs 2+1: w diff", len(wi), "z diff", len(zi))
