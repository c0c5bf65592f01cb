"""k_batch_chain on a C5 slice or the C2 sweep: us per iteration (one wave) and, with COT_TRACE=1, the per-phase
cycle breakdown of the chain CTA and the producers."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_13147_b200 as cot
import synthetic
wl = os.environ.get("WL", "C5"); B = int(os.environ.get("B", "22")); iters = int(os.environ.get("ITERS", "200"))
p = synthetic.c5_batched(B=B) if wl == "C5" else synthetic.c2_sweep()
dev = torch.device("cuda:0")
D = lambda x: torch.as_tensor(x, device=dev)
prob = cot.CerotProblem(D(p.C), D(p.alpha), D(p.beta), D(p.eps))
for rep in range(3):
    prob.init()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); prob.iterate(iters); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"{wl} B={p.B} iters={iters} path={cot.lib().cot_iter_path(p.B, p.n, p.m, 0, 0)} env="
      f"{ {k: v for k, v in os.environ.items() if k.startswith('COT_')} }: {ms*1e3/iters:.3f} us/iter, "
      f"{p.B*p.n*p.m*p.m*iters/ms/1e9:.3e} evals/s", flush=True)
