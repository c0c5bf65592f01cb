#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
{
for g in 8 4; do
  python scripts/ubench_fused.py --shard-alone $g --iters 400
  COT_WIDE=1 python scripts/ubench_fused.py --shard-alone $g --iters 400 | sed 's/^/wide /'
  COT_WIDE=1 python scripts/ubench_fused.py --shard-alone $g --iters 400 --flags 0x200 | sed 's/^/wide nosync /'
done
COT_WIDE=1 COT_TRACE=1 python scripts/ubench_fused.py --shard-alone 8 --iters 400 2>&1 | grep "cot trace" | tail -1
} > gpurun_out/shard_probe.log 2>&1
cat gpurun_out/shard_probe.log
