#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q -p no:cacheprovider 2>&1 | tail -2
for ws in 1 0; do
  echo "== COT_BATCH_WS=$ws"
  COT_BATCH_WS=$ws COT_TRACE=1 B=256 ITERS=100 python scripts/ubench_batch.py 2>&1 | grep trace | tail -1
  COT_BATCH_WS=$ws B=4096 ITERS=50 python scripts/ubench_batch.py
  COT_BATCH_WS=$ws python scripts/ubench_c2.py
done
