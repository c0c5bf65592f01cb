"""Microbenchmark of the persistent C-EROT kernel on C4: full kernel vs diagnostic variants (pure TMA
stream, compute without device-wide sync). Prints us/iteration and GB/s of the algorithmic C+G bytes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2311_13147_b200 as cot
import synthetic

p = synthetic.c3_image() if os.environ.get("WL") == "C3" else synthetic.c4_large(m=int(os.environ.get("M", "1024")), n=int(os.environ.get("N", "64")))
dev = torch.device("cuda:0")
C = torch.as_tensor(p.C, device=dev)
prob = cot.CerotProblem(C, torch.as_tensor(p.alpha, device=dev), torch.as_tensor(p.beta, device=dev), p.eps)
iters = int(os.environ.get("ITERS", "200"))
bytes_iter = (p.n + 1) * p.m * p.m * 4
variants = [("full", 0), ("no_sync", 0x200), ("no_compute", 0x100), ("stream_only", 0x300)]
for name, fl in variants:
    for rep in range(2):
        prob.init()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        prob.iterate(iters, flags=fl)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / iters
    print(f"{name:12s} {us:8.2f} us/iter  {bytes_iter / us / 1e3:8.1f} GB/s", flush=True)
