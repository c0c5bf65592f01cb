#!/bin/bash
# Chain latency vs streaming: the 8-way shard and C3 with the C stream on/off (COT_DIAG_NO_STREAM) and the
# k-sum compute on/off (COT_DIAG_NO_COMPUTE). Diagnostic timings only (results are wrong with these flags).
for f in 0 0x400 0x100 0x500; do
  python scripts/ubench_fused.py --shard-alone 8 --iters 400 --flags $f
done
for f in 0 0x400 0x100 0x500; do
  echo "C3 flags $f"; COT_TRACE=1 FLAGS=$f WL=C3 ITERS=400 python scripts/ubench_trace.py 2>&1 | tail -1 | cut -c1-220
done
