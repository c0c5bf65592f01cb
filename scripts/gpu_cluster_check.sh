#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q -p no:cacheprovider 2>&1 | tail -3
B=4096 ITERS=50 python scripts/ubench_batch.py
COT_TRACE=1 B=144 ITERS=200 python scripts/ubench_batch.py
