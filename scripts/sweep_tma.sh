timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for sb in 32768 65536; do for qn in 4 8; do
  echo "== SLOT_BYTES=$sb QN=$qn"; COT_QN=$qn COT_SLOT_BYTES=$sb ITERS=200 timeout 120 python scripts/ubench_iter.py 2>&1 | grep -E "full|no_sync|stream"
done; done
COT_TRACE=1 ITERS=100 timeout 120 python scripts/ubench_iter.py 2>&1 | grep trace | head -1
