# usage (under gpurun): bash scripts/gpu_round_measure.sh  -> gpurun_out/{bench_*.json, launches.csv, prof_iter.ncu-rep}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python bench.py > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; echo c4=$?
for w in C2 C2e2 C3; do timeout 600 python bench.py --workload $w --no-cpu > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w=$?; done
timeout 900 python bench.py --workload C5 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo C5=$?
COT_BENCH_MODE=precomputed timeout 600 python bench.py --no-cpu > gpurun_out/bench_C4_precomputed.json 2> gpurun_out/bench_pre.err; echo pre=$?
COT_BENCH_SHARDED=1 timeout 600 python bench.py --no-cpu > gpurun_out/bench_C4_fused1.json 2> gpurun_out/bench_f1.err; echo f1=$?
COT_SHARD_IMPL=nccl COT_BENCH_SHARDED=1 timeout 600 python bench.py --no-cpu > gpurun_out/bench_C4_nccl1.json 2> gpurun_out/bench_n1.err; echo n1=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
for g in 2 4 8; do timeout 120 python scripts/ubench_fused.py --shard-alone $g --iters 200 >> gpurun_out/shard_alone.jsonl 2>/dev/null; done
timeout 300 python scripts/ubench_fused.py >> gpurun_out/fused_emulated.jsonl 2>/dev/null
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
CMD2="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --iters 50"
timeout 300 $CMD2 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_iter_tma -s 1 -c 1 -o gpurun_out/prof_iter $CMD2 > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
for f in gpurun_out/bench_*.err; do echo $f; tail -2 $f; done
