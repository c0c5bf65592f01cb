# usage (under gpurun): bash scripts/ab.sh A.so B.so ...  -- alternates the libraries, 2 rounds each
for round in 1 2; do
  for lib in "$@"; do
    cp "$lib" paper_2311_13147_b200/libcyclicot.so
    touch paper_2311_13147_b200/libcyclicot.so
    s8=$(timeout 120 python scripts/ubench_fused.py --shard-alone 8 --iters 200 2>/dev/null | tail -1 | python -c "import json,sys; print('%.2f' % json.loads(sys.stdin.read())['us_per_iter'])")
    c3=$(WL=C3 ITERS=200 timeout 120 python scripts/ubench_iter.py 2>&1 | head -1 | awk '{print $2}')
    c4=$(N=64 ITERS=200 timeout 120 python scripts/ubench_iter.py 2>&1 | head -1 | awk '{print $2}')
    echo "round $round $lib: shard8 $s8 us  C3 $c3 us  C4 $c4 us"
  done
done
