#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
{
timeout 600 python -m pytest tests/test_gpu_dist.py -m gpu -q 2>&1 | tail -3
COT_SHARD_IMPL=nccl COT_BENCH_SHARDED=1 timeout 600 python bench.py --no-cpu --no-e2e --steps 3 --warmup 2 > gpurun_out/nccl1.json 2> gpurun_out/nccl1.err
COT_SHARD_GRAPH=0 COT_SHARD_IMPL=nccl COT_BENCH_SHARDED=1 timeout 600 python bench.py --no-cpu --no-e2e --steps 3 --warmup 2 > gpurun_out/nccl1_nograph.json 2> gpurun_out/nccl1_ng.err
for f in nccl1 nccl1_nograph; do python -c "import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['roofline']['us_per_iter'], d['exchange'], d['config']['parallelism'])" || tail -5 gpurun_out/$f.err; done
} > gpurun_out/nccl_check.log 2>&1
cat gpurun_out/nccl_check.log
