#!/bin/bash
# cluster-exchange chain microbenchmark sweep
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
{
for mode in 0 1; do
for cfg in "16 7" "8 15" "8 8" "16 2" "4 32" "16 1" "8 1"; do
  timeout 60 ./scripts/ubench/cxchain $cfg 1024 4000 190000 $mode
done
done
} > gpurun_out/cx.log 2>&1
cat gpurun_out/cx.log
