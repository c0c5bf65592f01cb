#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
{
for ms in 2 3 4; do
  for g in 8 4; do COT_MIN_SLOTS=$ms python scripts/ubench_fused.py --shard-alone $g --iters 400 | sed "s/^/ms=$ms /"; done
  COT_MIN_SLOTS=$ms python scripts/ubench_fused.py --ranks 1 --iters 200 | sed "s/^/ms=$ms /"
done
COT_MIN_SLOTS=2 python scripts/ubench_fused.py --shard-alone 4 --iters 400 --flags 0x200 | sed "s/^/ms=2 nosync /"
COT_MIN_SLOTS=2 python scripts/ubench_fused.py --shard-alone 8 --iters 400 --flags 0x200 | sed "s/^/ms=2 nosync /"
} > gpurun_out/shard_probe.log 2>&1
cat gpurun_out/shard_probe.log
