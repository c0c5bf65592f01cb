#!/bin/bash
# k-sum warps per row count in the warp-specialised cluster kernel (COT_BATCH_KR rows per k-sum warp).
COT_BATCH_KR=4 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "c5 or c2 or cluster or batch" 2>&1 | tail -1
for kr in 2 3 4; do
  echo "== KR=$kr"
  COT_BATCH_KR=$kr COT_TRACE=1 B=256 ITERS=100 python scripts/ubench_batch.py 2>&1 | grep trace | tail -1
  COT_BATCH_KR=$kr B=4096 ITERS=50 python scripts/ubench_batch.py
  COT_BATCH_KR=$kr python scripts/ubench_c2.py
done
