#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
{
python scripts/ubench_chain.py
COT_TRACE=1 ITERS=50 python scripts/ubench_chain.py 2>&1 | tail -2
WL=C2 python scripts/ubench_chain.py
WL=C2 COT_TRACE=1 ITERS=50 python scripts/ubench_chain.py 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "cluster or c2 or c5 or precomputed or chain or freeze" 2>&1 | tail -3
} > gpurun_out/chain_trace.log 2>&1
cat gpurun_out/chain_trace.log
