#!/bin/bash
# Round measurement pass (under gpurun): bench lines, shard/emulation timings, solve-to-tolerance lines, ncu launch
# lists and top-kernel captures -> gpurun_out/r02/
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/r02
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 900 python bench.py > $O/bench_C4.json 2> $O/bench_C4.err; echo c4=$?
for w in C2 C2e2 C3; do timeout 600 python bench.py --workload $w --no-cpu > $O/bench_$w.json 2> $O/bench_$w.err; echo $w=$?; done
timeout 900 python bench.py --workload C5 --steps 3 --warmup 3 --no-cpu > $O/bench_C5.json 2> $O/bench_C5.err; echo C5=$?
COT_BENCH_MODE=precomputed timeout 600 python bench.py --no-cpu > $O/bench_C4_precomputed.json 2> $O/bench_pre.err; echo pre=$?
COT_BENCH_FLAGS=0x10 timeout 600 python bench.py --no-cpu > $O/bench_C4_deterministic.json 2> $O/bench_det.err; echo det=$?
COT_BENCH_SHARDED=1 timeout 600 python bench.py --no-cpu > $O/bench_C4_fused1.json 2> $O/bench_f1.err; echo f1=$?
COT_SHARD_IMPL=nccl COT_BENCH_SHARDED=1 timeout 600 python bench.py --no-cpu > $O/bench_C4_nccl1.json 2> $O/bench_n1.err; echo n1=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_ref.err; echo ref=$?
for g in 2 4 8; do timeout 120 python scripts/ubench_fused.py --shard-alone $g --iters 400 >> $O/shard_alone.jsonl 2>/dev/null; done
timeout 300 python scripts/ubench_fused.py >> $O/fused_emulated.jsonl 2>/dev/null
timeout 300 python scripts/bench_solve.py > $O/solve_to_tol.jsonl 2> $O/solve.err
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/C4_launches.csv $CMD > $O/ncu_launch.log 2>&1; echo ncu1=$?
CMD5="python bench.py --workload C5 --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 300 $CMD5 > $O/plain5.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/C5_launches.csv $CMD5 > $O/ncu_launch5.log 2>&1; echo ncu5=$?
CMD2="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --iters 50"
timeout 300 $CMD2 > $O/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_iter_tma -s 1 -c 1 -o $O/C4_iter_prof $CMD2 > $O/ncu_full.log 2>&1; echo ncu2=$?
CMD3="python scripts/ubench_chain.py"
timeout 300 $CMD3 > $O/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_batch_chain -s 2 -c 1 -o $O/C5_chain_prof $CMD3 > $O/ncu_full3.log 2>&1; echo ncu3=$?
for f in $O/bench_*.err; do echo $f; tail -2 $f; done
