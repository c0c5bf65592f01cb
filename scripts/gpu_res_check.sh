#!/bin/bash
# K-ITER-RES check: shard-alone timings (resident vs streaming kernel) with the per-phase trace, C3, parity subsets.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
{
for g in 8 4; do
  timeout 120 python scripts/ubench_fused.py --shard-alone $g --iters 400 | sed "s/^/res /"
  COT_RES_THROTTLE=0 timeout 120 python scripts/ubench_fused.py --shard-alone $g --iters 400 | sed "s/^/res nothrottle /"
  COT_RES_THROTTLE=1 timeout 120 python scripts/ubench_fused.py --shard-alone $g --iters 400 | sed "s/^/res throttle /"
  COT_TRACE=1 timeout 120 python scripts/ubench_fused.py --shard-alone $g --iters 400 2>&1 | grep "res trace" | tail -1
done
timeout 300 python bench.py --workload C3 --steps 3 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', d['roofline']['us_per_iter'], d['roofline']['kernel'][:40], d['roofline']['frac'])"
WL=C3 COT_TRACE=1 timeout 300 python scripts/ubench_iter.py 2>&1 | grep -E "res trace|full" | head -2
} > gpurun_out/res_check.log 2>&1
timeout 900 python -m pytest tests/test_gpu_res.py tests/test_gpu_fused.py -q -x > gpurun_out/res_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/res_tests.log
cat gpurun_out/res_check.log; grep -E "passed|failed|FAILED|Error" gpurun_out/res_tests.log | head -30
