#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
CMD="python scripts/ubench_fused.py --shard-alone 4 --iters 100 --flags 0x200"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_iter_tma -s 1 -c 1 -f -o gpurun_out/tma_prof $CMD > gpurun_out/ncu_tma.log 2>&1
echo rc=$?; tail -2 gpurun_out/ncu_tma.log
