#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
{
for g in 8 4 2; do
  python scripts/ubench_fused.py --shard-alone $g --iters 400
  COT_CLAYOUT=rnm python scripts/ubench_fused.py --shard-alone $g --iters 400 | sed 's/^/rnm /'
  COT_CLAYOUT=rnm python scripts/ubench_fused.py --shard-alone $g --iters 400 --flags 0x300 | sed 's/^/rnm stream-only /'
  python scripts/ubench_fused.py --shard-alone $g --iters 400 --flags 0x300 | sed 's/^/stream-only /'
done
} > gpurun_out/shard_probe.log 2>&1
cat gpurun_out/shard_probe.log
