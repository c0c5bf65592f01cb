#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
{
python scripts/ubench_chain.py
COT_CHAIN_DIAG=1 python scripts/ubench_chain.py
COT_CHAIN_DIAG=2 python scripts/ubench_chain.py
WL=C2 python scripts/ubench_chain.py
WL=C2 COT_CHAIN_DIAG=1 python scripts/ubench_chain.py
WL=C2 COT_CHAIN_DIAG=2 python scripts/ubench_chain.py
} > gpurun_out/chain_trace.log 2>&1
cat gpurun_out/chain_trace.log
