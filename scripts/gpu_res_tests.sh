#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_res.py tests/test_gpu_memsafety.py tests/test_gpu_fused.py -q -x > gpurun_out/res_tests2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/res_tests2.log
tail -30 gpurun_out/res_tests2.log
