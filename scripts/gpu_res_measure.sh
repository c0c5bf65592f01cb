#!/bin/bash
# K-ITER-RES measurement pass (under gpurun) -> gpurun_out/r02r/: C3 bench line on the resident kernel (and on the
# streaming one for comparison), the 8-/4-/2-way C4 shards alone (resident vs streaming), solve-to-tolerance,
# the C3 ncu launch list, ncu --set full of k_iter_res (C3 and the 1/8 shard) with per-line stall reasons
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/r02r
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 600 python bench.py --workload C3 --no-cpu > $O/bench_C3.json 2> $O/bench_C3.err; echo C3=$?
COT_RES=0 timeout 600 python bench.py --workload C3 --no-cpu > $O/bench_C3_tma.json 2> $O/bench_C3_tma.err; echo C3tma=$?
for g in 8 4 2; do
  timeout 120 python scripts/ubench_fused.py --shard-alone $g --iters 400 | sed 's/"mode"/"kernel": "res (default)", "mode"/' >> $O/shard_alone.jsonl 2>/dev/null
  COT_RES=0 timeout 120 python scripts/ubench_fused.py --shard-alone $g --iters 400 | sed 's/"mode"/"kernel": "tma (COT_RES=0)", "mode"/' >> $O/shard_alone.jsonl 2>/dev/null
done
for hh in 1 2 4; do
  COT_RES_H=$hh timeout 120 python scripts/ubench_fused.py --shard-alone 8 --iters 400 | sed "s/\"mode\"/\"kernel\": \"res h=$hh\", \"mode\"/" >> $O/shard_alone.jsonl 2>/dev/null
done
for g in 8 4; do COT_TRACE=1 timeout 120 python scripts/ubench_fused.py --shard-alone $g --iters 400 2>&1 | grep "res trace" | sed "s/^/1_of_$g /" >> $O/res_trace.txt; done
WL=C3 COT_TRACE=1 timeout 300 python scripts/ubench_iter.py 2>&1 | grep "res trace" | head -1 | sed "s/^/C3 /" >> $O/res_trace.txt
timeout 300 python scripts/bench_solve.py > $O/solve_to_tol.jsonl 2> $O/solve.err
CMD="python bench.py --workload C3 --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/C3_launches.csv $CMD > $O/ncu_launch.log 2>&1; echo ncu1=$?
WL=C3 ITERS=60 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_iter_res -c 1 -o $O/C3_res_prof python scripts/ubench_iter.py > $O/ncu_c3.log 2>&1; echo ncu_c3=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_iter_res -c 1 -o $O/C4s8_res_prof python scripts/ubench_fused.py --shard-alone 8 --iters 60 > $O/ncu_c4s8.log 2>&1; echo ncu_c4s8=$?
python scripts/ncu_stall_lines.py $O/C3_res_prof.ncu-rep 40 > $O/C3_res_stall_lines.txt 2>&1
python scripts/ncu_stall_lines.py $O/C4s8_res_prof.ncu-rep 40 > $O/C4s8_res_stall_lines.txt 2>&1
ncu -i $O/C3_res_prof.ncu-rep --page raw --csv > $O/C3_res_raw.csv 2>/dev/null
ncu -i $O/C4s8_res_prof.ncu-rep --page raw --csv > $O/C4s8_res_raw.csv 2>/dev/null
rm -f $O/*.ncu-rep
cat $O/shard_alone.jsonl; cat $O/res_trace.txt; for f in $O/bench_*.err; do echo $f; tail -2 $f; done
