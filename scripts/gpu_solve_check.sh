#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
{
./scripts/ubench/gc_test
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_deterministic.py -m gpu -q -k "solve or boundaries or c1 or freeze" 2>&1 | tail -15
python scripts/bench_solve.py
} > gpurun_out/solve_check.log 2>&1
cat gpurun_out/solve_check.log
