timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for vec in 4 2; do for sb in 16384 32768 65536; do
  echo "== VEC=$vec SLOT_BYTES=$sb"; COT_VEC=$vec COT_SLOT_BYTES=$sb ITERS=200 python scripts/ubench_iter.py 2>&1 | grep -E "full|stream_only|no_sync"
done; done
COT_TRACE=1 ITERS=100 python scripts/ubench_iter.py 2>&1 | grep trace | head -1
