#!/bin/bash
# C4 default line after the TMEM-resident k-blocks: the driver's bench command, launch list, ncu --set full of
# k_iter_tma (50 iterations), summaries -> gpurun_out/r02t/
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/r02u; mkdir -p $O
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_C4.json 2> $O/bench_C4.err; echo c4=$?
COT_KTM=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > $O/bench_C4_ktm0.json 2> $O/bench_C4_ktm0.err; echo c4k0=$?
COT_BENCH_FLAGS=0x10 timeout 600 python bench.py --no-cpu > $O/bench_C4_deterministic.json 2> $O/bench_det.err; echo det=$?
COT_BENCH_SHARDED=1 timeout 600 python bench.py --no-cpu > $O/bench_C4_fused1.json 2> $O/bench_f1.err; echo f1=$?
timeout 300 python scripts/ubench_fused.py --iters 200 --ranks 1,2,4,8 > $O/fused_emulated.jsonl 2>/dev/null; echo emu=$?
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/C4_launches.csv $CMD > $O/ncu_launch.log 2>&1; echo ncu1=$?
CMD2="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --iters 50"
timeout 300 $CMD2 > $O/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_iter_tma -s 1 -c 1 -o $O/C4_iter_prof $CMD2 > $O/ncu_full.log 2>&1; echo ncu2=$?
python scripts/summarize_ncu.py r02u C4 $O/C4_launches.csv $O/C4_iter_prof.ncu-rep 50 > $O/summ.log 2>&1; echo summ=$?
python scripts/ncu_stall_lines.py $O/C4_iter_prof.ncu-rep 30 > $O/C4_iter_stall_lines.txt 2>&1
rm -f $O/*.ncu-rep
cat $O/summ.log | tail -5; cat $O/fused_emulated.jsonl
