import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2311_13147_b200 as cot, synthetic, oracle
dev = torch.device("cuda:0")
for name, p in [("C2", synthetic.c2_ring(eps_factor=0.1)), ("C4m256", synthetic.c4_large(m=256, n=16))]:
    for iters in (1, 2, 3):
        out = {}
        for path, fl in (("tma", 0), ("ldg", cot.COT_FORCE_LDG)):
            prob = cot.CerotProblem(torch.as_tensor(p.C, device=dev), torch.as_tensor(p.alpha, device=dev),
                                    torch.as_tensor(p.beta, device=dev), p.eps)
            prob.init().iterate(iters, flags=fl)
            torch.cuda.synchronize()
            out[path] = (prob.w_hat.cpu().numpy(), prob.z_hat.cpu().numpy())
            try:
                print(name, iters, path, prob.state())
            except Exception as e:
                print(name, iters, path, "state error", e)
        dw = np.abs(out["tma"][0] - out["ldg"][0]); dz = np.abs(out["tma"][1] - out["ldg"][1])
        print(f"  {name} iters={iters} max|dw|={dw.max():.3e} at {dw.argmax()} max|dz|={dz.max():.3e} at {dz.argmax()}")
        print("   w tma", out["tma"][0][:4], "ldg", out["ldg"][0][:4])
        print("   z tma", out["tma"][1][:4], "ldg", out["ldg"][1][:4])
