"""Small runs of every kernel of libcyclicot through the C ABI, one case per process, for compute-sanitizer
(scripts/gpu_sanitize.sh runs each case under one tool: memcheck, racecheck, synccheck or initcheck).

  python scripts/sanitize_cases.py --list
  python scripts/sanitize_cases.py --case NAME
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthetic  # noqa: E402
import paper_2311_13147_b200 as cot  # noqa: E402
from paper_2311_13147_b200 import dist as cdist  # noqa: E402

DEV = torch.device("cuda:0")
D = lambda x: torch.as_tensor(np.ascontiguousarray(x), device=DEV)  # noqa: E731


def _iterate(p, iters, flags=0, plan=True):
    prob = cot.CerotProblem(D(p.C), D(p.alpha), D(p.beta), D(p.eps)).init()
    prob.iterate(iters, flags=flags)
    if plan:
        prob.plan(T_blocks=True)
    torch.cuda.synchronize()
    prob.state()


def case_aggregate():       # k_aggregate (fp32 and fp64)
    cot.clot_aggregate(D(synthetic.c2_ring().C))
    cot.clot_aggregate(D(synthetic.c1_tiny().C))


def case_expand_rows():     # k_expand_rows (C5 shape), both modes
    rng = np.random.default_rng(1)
    T = rng.random((2, 16, 128, 128)).astype(np.float32)
    cot.clot_expand(D(T), 16)
    S = rng.random((2, 128, 128)).astype(np.float32)
    A = rng.integers(0, 16, size=(2, 128, 128)).astype(np.int32)
    cot.clot_expand(D(S), 16, argmin=D(A))


def case_expand_bulk():     # k_expand_bulk (m*4 % 16 == 0, rows too large for k_expand_rows), both modes
    rng = np.random.default_rng(2)
    T = rng.random((7, 512, 512)).astype(np.float32)
    assert cot.lib().cot_expand_path(7, 512, 0) == 1
    cot.clot_expand(D(T), 7)
    A = rng.integers(0, 7, size=(512, 512)).astype(np.int32)
    cot.clot_expand(D(T[0]), 7, argmin=D(A))


def case_expand_generic():  # k_expand (ragged m)
    rng = np.random.default_rng(3)
    T = rng.random((3, 37, 37)).astype(np.float32)
    cot.clot_expand(D(T), 3)


def case_ldg_fp64():        # k_rows_ldg + k_cols (fp64 C1), plan
    _iterate(synthetic.c1_tiny(), 5)


def case_chain():           # k_batch_chain (C2 sweep: three problems, 8-CTA clusters)
    _iterate(synthetic.c2_sweep(), 5)


def case_chain_batch():     # k_batch_chain, 6-CTA clusters (more problems than one wave of 8-CTA clusters)
    _iterate(synthetic.c5_batched(B=24), 3)


def case_cluster_ws():      # k_batch_cluster_ws (COT_BATCH_CHAIN=0, m <= 128)
    os.environ["COT_BATCH_CHAIN"] = "0"
    _iterate(synthetic.c2_ring(), 5)


def case_cluster_interleaved():   # k_batch_cluster (m > 128)
    _iterate(synthetic.random_cyclic(seed=4, n=3, m=192, dtype=np.float32, eps=0.05, B=2), 4)


def case_tma_small():       # k_iter_tma forced on a small problem (ring, queue, LL lines, resident k-blocks)
    _iterate(synthetic.random_cyclic(seed=5, n=9, m=256, dtype=np.float32, eps=0.05), 4, flags=cot.COT_FORCE_TMA)


def case_tma_c3():          # k_iter_tma on C3 (row-per-warp epilogue)
    _iterate(synthetic.c3_image(), 3)


def case_tma_deterministic():   # k_iter_tma, COT_DETERMINISTIC (128-bit fixed-point partials)
    _iterate(synthetic.c4_large(m=256, n=8), 3, flags=cot.COT_DETERMINISTIC)


def case_precomputed():     # k_precompute + the row kernels with n = 1
    p = synthetic.c2_ring()
    prob = cot.CerotProblem(D(p.C), D(p.alpha), D(p.beta), D(p.eps)).init()
    prob.precompute()
    prob.iterate_precomputed(4)
    torch.cuda.synchronize()


def case_fused_emulated():  # k_iter_tma_emu: 2 emulated ranks, in-kernel exchange
    p = synthetic.c4_large(m=256, n=8)
    shards = []
    for r in range(2):
        b0, R = cdist.row_partition(p.m, 2, r)
        shards.append(cdist.ShardedCerot(D(p.C[:, b0:b0 + R, :]), D(p.alpha), D(p.beta), float(p.eps[0]), b0,
                                         p.m).init())
    xb = cdist.emulate_fused(shards, 3)
    torch.cuda.synchronize()
    cdist.free_xbufs(xb)


def case_sharded_split():   # rows-only launch + k_colsum + k_zupdate (the NCCL path without a communicator)
    p = synthetic.c4_large(m=256, n=8)
    sh = cdist.ShardedCerot(D(p.C), D(p.alpha), D(p.beta), float(p.eps[0]), 0, p.m).init()
    sh.iterate(3)
    sh.plan(T_local=True)
    torch.cuda.synchronize()


def case_two_stage():       # k_fold, k_tile, k_transpose_blocks, k_full_pass, k_full_finalize
    p = synthetic.random_cyclic(seed=6, n=4, m=32, dtype=np.float32, eps=0.1)
    a, b = synthetic.approx_symmetric(p)
    cot.two_stage_sinkhorn(D(a), D(b), D(p.C), 0.1, 3, 3)
    torch.cuda.synchronize()


def case_srot():            # k_srot sweeps + plan
    p = synthetic.random_cyclic(seed=7, n=4, m=32, dtype=np.float32, eps=0.1)
    cot.csrot_solve(D(p.C), D(p.alpha), D(p.beta), 0.5, max_sweeps=3, T_blocks=True)
    torch.cuda.synchronize()


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case")
    ap.add_argument("--list", action="store_true")
    a = ap.parse_args()
    if a.list:
        print(" ".join(CASES))
        return
    from paper_2311_13147_b200 import build
    build.build()
    cot.use_current_device()
    CASES[a.case]()
    torch.cuda.synchronize()
    print(f"case {a.case}: done")


if __name__ == "__main__":
    main()
