# usage (under gpurun): bench in every mode on one GPU -> gpurun_out/bench_*.json
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4=$?
COT_BENCH_SHARDED=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4_sharded1.json 2> gpurun_out/bench_c4_sharded1.err; echo sharded=$?
timeout 600 torchrun --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29577 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4_torchrun1.json 2> gpurun_out/bench_c4_torchrun1.err; echo torchrun=$?
for w in C2 C3; do timeout 600 python bench.py --steps 3 --warmup 3 --workload $w --no-cpu > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w=$?; done
COT_C5_B=1024 timeout 900 python bench.py --steps 3 --warmup 3 --workload C5 --no-cpu > gpurun_out/bench_C5_1024.json 2> gpurun_out/bench_C5.err; echo C5=$?
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
for f in gpurun_out/bench_*.err; do tail -2 $f; done
