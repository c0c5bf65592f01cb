#!/bin/bash
# What the driver runs at round end: the -m gpu suite, smoke(), and the default bench line (N=1, 20 steps)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
bash scripts/gpu_tests.sh
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench rc=$?"; wc -l gpurun_out/bench_default.json
python -c "import json; d=json.loads(open('gpurun_out/bench_default.json').read()); print(d['value'], d['roofline']['us_per_iter'], d['roofline']['frac'], d['clocks'], d['e2e']['value'], d['cpu_baseline']['value'], d['exchange'])"
