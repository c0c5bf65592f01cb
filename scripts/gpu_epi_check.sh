#!/bin/bash
# Parity of the persistent kernel + timing of the latency-bound and HBM-bound configurations.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_dist.py -x -q -p no:cacheprovider 2>&1 | tail -4
WL=C3 ITERS=400 python scripts/ubench_iter.py 2>&1 | head -2
ITERS=200 python scripts/ubench_iter.py 2>&1 | head -2
python scripts/ubench_fused.py --shard-alone 8 --iters 400
python scripts/ubench_fused.py --shard-alone 4 --iters 400
COT_TRACE=1 python scripts/ubench_fused.py --shard-alone 8 --iters 400 2>&1 | tail -2
COT_TRACE=1 WL=C3 ITERS=400 python scripts/ubench_trace.py 2>&1 | tail -1
