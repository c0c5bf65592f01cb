#!/bin/bash
# the fused path over NCCL symmetric memory: the single-rank test, and the bench line at one rank (C4 whole
# problem through cerot_iter_fused) for the IPC mapping, the NCCL window mapping and the NCCL split baseline
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/r02n
timeout 600 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -15
for impl in fused ncclwin nccl; do
  COT_SHARD_IMPL=$impl COT_BENCH_SHARDED=1 timeout 600 python bench.py --no-cpu > gpurun_out/r02n/bench_C4_$impl.json 2> gpurun_out/r02n/bench_C4_$impl.err
  python -c "import json; d=json.loads(open('gpurun_out/r02n/bench_C4_$impl.json').read()); print('$impl', d['roofline']['us_per_iter'], d['value'], d['exchange'])"
  tail -2 gpurun_out/r02n/bench_C4_$impl.err
done
