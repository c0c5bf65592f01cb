#!/bin/bash
# ncu --set full of k_batch_chain on one C5 wave (22 problems x 200 iterations)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
CMD="python scripts/ubench_chain.py"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_batch_chain -s 2 -c 1 -f \
    -o gpurun_out/chain_prof $CMD > gpurun_out/ncu_chain.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu_chain.log
