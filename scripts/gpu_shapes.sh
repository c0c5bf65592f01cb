#!/bin/bash
# Cluster shapes of the batched kernel: parity (the C5/C2 tests) and C5 / C2 timing per shape.
for sh in ${SHAPES:-0 1 2 3}; do
  echo "== shape $sh"
  COT_BATCH_SHAPE=$sh timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "c5 or c2 or batch or ring" 2>&1 | tail -1
  COT_BATCH_SHAPE=$sh B=4096 ITERS=50 python scripts/ubench_batch.py
  COT_BATCH_SHAPE=$sh COT_TRACE=1 B=256 ITERS=100 python scripts/ubench_batch.py 2>&1 | grep trace | tail -1
done
