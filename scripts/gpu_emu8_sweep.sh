# emulated 8-rank fused launch: L2 evict_last rows per virtual rank (COT_EVICT_LAST_ROWS) sweep
mkdir -p gpurun_out
: > gpurun_out/emu8.jsonl
for E in none 0 16 27 40; do
  if [ $E = none ]; then unset COT_EVICT_LAST_ROWS; else export COT_EVICT_LAST_ROWS=$E; fi
  echo "{\"evict_last_rows\": \"$E\"}" >> gpurun_out/emu8.jsonl
  timeout 300 python scripts/ubench_fused.py --ranks 8 >> gpurun_out/emu8.jsonl 2>> gpurun_out/emu8.err
done
