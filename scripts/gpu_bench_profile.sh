# usage (under gpurun): bash scripts/gpu_bench_profile.sh  -> gpurun_out/{pytest_gpu.log,bench_default.json,launches.csv,prof_iter.ncu-rep}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo rc=$?
tail -3 gpurun_out/bench_default.err
cat gpurun_out/bench_default.json
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 6 -c 6 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
CMD2="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --iters 50"
timeout 300 $CMD2 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_iter_tma -s 1 -c 1 -o gpurun_out/prof_iter $CMD2 > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
