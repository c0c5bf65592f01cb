mkdir -p gpurun_out
for E in default 0 150 300; do
  if [ $E = default ]; then unset COT_EVICT_LAST_ROWS; else export COT_EVICT_LAST_ROWS=$E; fi
  COT_SHARD_IMPL=nccl COT_BENCH_SHARDED=1 timeout 600 python bench.py --no-cpu > gpurun_out/n1_el_$E.json 2>> gpurun_out/n1_el.err; echo $E=$?
done
