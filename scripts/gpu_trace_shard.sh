#!/bin/bash
# Per-phase cycle traces of the latency-bound configurations (8-way C4 shard alone, C3).
set -x
export COT_TRACE=1
python scripts/ubench_fused.py --shard-alone 8 --iters 400
python scripts/ubench_fused.py --shard-alone 4 --iters 400
WL=C3 ITERS=400 python scripts/ubench_trace.py
