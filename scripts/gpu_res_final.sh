#!/bin/bash
# Final round-2 lines for k_iter_res after the count-byte rank-local level -> gpurun_out/r02f/
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/r02f; mkdir -p $O
for g in 8 4 2; do
  timeout 120 python scripts/ubench_fused.py --shard-alone $g --iters 400 | sed 's/"mode"/"kernel": "default", "mode"/' >> $O/shard_alone.jsonl 2>/dev/null
  COT_RES=0 timeout 120 python scripts/ubench_fused.py --shard-alone $g --iters 400 | sed 's/"mode"/"kernel": "k_iter_tma (COT_RES=0)", "mode"/' >> $O/shard_alone.jsonl 2>/dev/null
done
for hh in 1 2 4; do
  COT_RES_H=$hh timeout 120 python scripts/ubench_fused.py --shard-alone 8 --iters 400 | sed "s/\"mode\"/\"kernel\": \"k_iter_res h=$hh\", \"mode\"/" >> $O/shard_alone.jsonl 2>/dev/null
done
for g in 8 4; do COT_TRACE=1 timeout 120 python scripts/ubench_fused.py --shard-alone $g --iters 400 2>&1 | grep "res trace" | sed "s/^/1_of_$g /" >> $O/res_trace.txt; done
WL=C3 COT_TRACE=1 timeout 300 python scripts/ubench_iter.py 2>&1 | grep "res trace" | head -1 | sed "s/^/C3 /" >> $O/res_trace.txt
timeout 600 python bench.py --workload C3 --no-cpu > $O/bench_C3.json 2> $O/bench_C3.err; echo C3=$?
timeout 300 python scripts/ubench_fused.py --iters 200 --ranks 1,2,4,8 > $O/fused_emulated.jsonl 2>/dev/null; echo emu=$?
timeout 300 python scripts/bench_solve.py > $O/solve_to_tol.jsonl 2> $O/solve.err
cat $O/shard_alone.jsonl; cat $O/res_trace.txt
