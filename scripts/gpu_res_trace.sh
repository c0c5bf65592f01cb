#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for g in 8 4; do
  timeout 120 python scripts/ubench_fused.py --shard-alone $g --iters 400
  COT_TRACE=1 timeout 120 python scripts/ubench_fused.py --shard-alone $g --iters 400 2>&1 | grep "res trace" | tail -1
done
timeout 900 python -m pytest tests/test_gpu_res.py tests/test_gpu_fused.py tests/test_gpu_memsafety.py -q -x 2>&1 | tail -3
