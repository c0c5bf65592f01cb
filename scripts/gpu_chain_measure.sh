#!/bin/bash
# Chain-kernel measurement pass (under gpurun): the full -m gpu suite, the C5 / C2 bench lines, the C5 launch list
# and one ncu --set full capture of k_batch_chain -> gpurun_out/r02c/
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/r02c
mkdir -p $O
python -c "from paper_2311_13147_b200 import build as b; b.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/gpu_tests.log 2>&1; echo tests=$?
tail -3 $O/gpu_tests.log
timeout 900 python bench.py --workload C5 --steps 3 --warmup 3 --no-cpu > $O/bench_C5.json 2> $O/bench_C5.err; echo C5=$?
for w in C2 C2e2; do timeout 600 python bench.py --workload $w --no-cpu > $O/bench_$w.json 2> $O/bench_$w.err; echo $w=$?; done
CMD5="python bench.py --workload C5 --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 300 $CMD5 > $O/plain5.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/C5_launches.csv $CMD5 > $O/ncu_launch5.log 2>&1; echo ncu5=$?
CMD3="python scripts/ubench_chain.py"
timeout 300 $CMD3 > $O/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_batch_chain -s 2 -c 1 -o $O/C5_chain_prof $CMD3 > $O/ncu_full3.log 2>&1; echo ncu3=$?
COT_TRACE=1 ITERS=400 python scripts/ubench_chain.py > $O/trace.log 2>&1
