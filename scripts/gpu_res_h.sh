cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for hh in 1 2 4; do COT_RES_H=$hh WL=C3 COT_TRACE=1 timeout 120 python scripts/ubench_iter.py 2>&1 | grep -E "res trace|full" | head -2 | sed "s/^/C3 h$hh /"; done
timeout 120 python scripts/ubench_fused.py --shard-alone 8 --iters 400
timeout 120 python scripts/ubench_fused.py --shard-alone 4 --iters 400
