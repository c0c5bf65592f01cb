# usage (under gpurun): WL=C3|N=.. bash scripts/ncu_iter.sh <tag>  -> gpurun_out/prof_<tag>.ncu-rep (+ csv pages)
set -x
TAG=${1:-iter}
ITERS=${ITERS:-30} timeout 300 python scripts/ubench_one.py > gpurun_out/plain_$TAG.log 2>&1 || exit 1
ITERS=${ITERS:-30} timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_iter_tma -s 1 -c 1 \
  -o gpurun_out/prof_$TAG python scripts/ubench_one.py > gpurun_out/ncu_$TAG.log 2>&1; echo ncu=$?
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv 2>/dev/null
ls -la gpurun_out/
