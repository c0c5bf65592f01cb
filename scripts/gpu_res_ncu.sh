#!/bin/bash
# ncu --set full of one k_iter_res launch: C3 (200 iterations) and the 1/8 C4 shard (fused, one rank)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
ITERS=60 WL=C3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_iter_res -c 1 -o $O/C3_res WL=C3 python scripts/ubench_iter.py > $O/ncu_c3.log 2>&1; echo ncu_c3=$?
WL=C3 ITERS=60 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_iter_res -c 1 -o $O/C3_res python scripts/ubench_iter.py > $O/ncu_c3.log 2>&1; echo ncu_c3=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_iter_res -c 1 -o $O/C4s8_res python scripts/ubench_fused.py --shard-alone 8 --iters 60 > $O/ncu_c4s8.log 2>&1; echo ncu_c4s8=$?
python scripts/ncu_stall_lines.py $O/C3_res.ncu-rep 40 > $O/C3_stall_lines.txt 2>&1
python scripts/ncu_stall_lines.py $O/C4s8_res.ncu-rep 40 > $O/C4s8_stall_lines.txt 2>&1
head -50 $O/C3_stall_lines.txt
