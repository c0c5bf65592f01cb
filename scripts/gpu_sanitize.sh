#!/bin/bash
# usage (under gpurun): bash scripts/gpu_sanitize.sh TOOL   (TOOL = plain | memcheck | racecheck | synccheck | initcheck)
# ONE compute-sanitizer tool per gpurun call (B200_PROFILING.md). Each kernel case runs in its own process with its
# own timeout; logs in gpurun_out/sanitizer_r02/TOOL_CASE.log, one summary line per case in TOOL_summary.txt.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
TOOL=${1:-plain}
OUT=gpurun_out/sanitizer_r02
mkdir -p $OUT
CASES=$(python scripts/sanitize_cases.py --list)
: > $OUT/${TOOL}_summary.txt
for c in $CASES; do
  if [ "$TOOL" = plain ]; then
    timeout 300 python scripts/sanitize_cases.py --case $c > $OUT/plain_$c.log 2>&1
    echo "$c rc=$?" >> $OUT/plain_summary.txt
  else
    timeout ${CASE_TIMEOUT:-600} /usr/local/cuda/bin/compute-sanitizer --tool $TOOL --kernel-regex kns=cot \
      --print-limit 20 python scripts/sanitize_cases.py --case $c > $OUT/${TOOL}_$c.log 2>&1
    rc=$?
    echo "$c rc=$rc $(grep -h 'ERROR SUMMARY\|LEAK SUMMARY\|RACECHECK SUMMARY' $OUT/${TOOL}_$c.log | tr '\n' ' ')" >> $OUT/${TOOL}_summary.txt
  fi
done
cat $OUT/${TOOL}_summary.txt
