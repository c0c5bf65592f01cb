#!/bin/bash
# K-ITER-RES check: shard-alone timings (resident vs streaming kernel) with the per-phase trace, C3, parity subsets.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
{
for hh in 1 2 4; do
  COT_RES_H=$hh timeout 120 python scripts/ubench_fused.py --shard-alone 8 --iters 400 | sed "s/^/res h$hh /"
  COT_TRACE=1 COT_RES_H=$hh timeout 120 python scripts/ubench_fused.py --shard-alone 8 --iters 400 2>&1 | grep "res trace" | tail -1
done
timeout 120 python scripts/ubench_fused.py --shard-alone 4 --iters 400 | sed 's/^/res /'
timeout 300 python bench.py --workload C3 --steps 3 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', d['roofline']['us_per_iter'], d['roofline']['kernel'][:40], d['roofline']['frac'])"
WL=C3 COT_TRACE=1 timeout 300 python scripts/ubench_iter.py 2>&1 | grep -E "res trace|full" | head -3
} > gpurun_out/res_check.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -q > gpurun_out/res_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/res_tests.log
cat gpurun_out/res_check.log; grep -E "passed|failed|FAILED|Error" gpurun_out/res_tests.log | head -30
