"""One traced persistent launch (COT_TRACE=1 prints the per-phase cycle breakdown), FLAGS selectable."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["COT_TRACE"] = "1"
import torch
import paper_2311_13147_b200 as cot
import synthetic
p = synthetic.c3_image() if os.environ.get("WL") == "C3" else synthetic.c4_large(m=int(os.environ.get("M", "1024")), n=int(os.environ.get("N", "64")))
dev = torch.device("cuda:0")
prob = cot.CerotProblem(torch.as_tensor(p.C, device=dev), torch.as_tensor(p.alpha, device=dev),
                        torch.as_tensor(p.beta, device=dev), p.eps)
prob.init().iterate(int(os.environ.get("ITERS", "200")), flags=int(os.environ.get("FLAGS", "0"), 0))
torch.cuda.synchronize()
