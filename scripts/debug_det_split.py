import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthetic, paper_2311_13147_b200 as cot
dev = torch.device("cuda:0"); D = lambda x: torch.as_tensor(np.ascontiguousarray(x), device=dev)
for name, p in (("C3", synthetic.c3_image()),):
    def run(split, flags=cot.COT_DETERMINISTIC):
        prob = cot.CerotProblem(D(p.C), D(p.alpha), D(p.beta), D(p.eps)).init()
        for k in split: prob.iterate(k, flags=flags)
        torch.cuda.synchronize()
        return prob.w_hat.cpu().numpy(), prob.z_hat.cpu().numpy()
    w0, z0 = run([25])
    for split in ([25], [7, 11, 7], [12, 13], [5, 20], [20, 5]):
        w, z = run(split)
        dz = np.nonzero(z.view(np.uint64) != z0.view(np.uint64))[0]
        dw = np.nonzero(w.view(np.uint64) != w0.view(np.uint64))[0]
        print(name, split, "z diff", len(dz), dz[:8], np.abs(z - z0).max(), "w diff", len(dw), dw[:8], np.abs(w - w0).max())
