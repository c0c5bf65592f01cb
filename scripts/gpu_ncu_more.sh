# usage (under gpurun): bash scripts/gpu_ncu_more.sh -> gpurun_out/{launches_C3.csv,prof_C3.ncu-rep,launches_C5.csv,prof_C5.ncu-rep}
set -x
for w in C3 C5; do
  K=$([ $w = C5 ] && echo k_batch_cluster || echo k_iter_tma)
  CMD="python bench.py --workload $w --steps 1 --warmup 1 --no-cpu --no-e2e"
  timeout 600 $CMD > gpurun_out/plain_$w.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$w.csv $CMD > gpurun_out/ncu_launch_$w.log 2>&1; echo ncu1_$w=$?
  CMD2="python bench.py --workload $w --steps 1 --warmup 1 --no-cpu --no-e2e --iters 50"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/prof_$w $CMD2 > gpurun_out/ncu_full_$w.log 2>&1; echo ncu2_$w=$?
done
