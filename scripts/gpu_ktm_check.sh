#!/bin/bash
# k_iter_tma with TMEM-resident k-blocks (ktm) vs without (COT_KTM=0): C4 iteration timing, bench line, parity
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for kt in 0 100; do COT_KTM=$kt ITERS=200 timeout 300 python scripts/ubench_iter.py 2>&1 | grep full | sed "s/^/C4 ktm<=$kt /"; done
COT_KTM=0 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('bench ktm0', d['value'], r['us_per_iter'], r['frac'], d['clocks']['sm_mhz'])"
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('bench ktm', d['value'], r['us_per_iter'], r['frac'], d['clocks']['sm_mhz'])"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_deterministic.py tests/test_gpu_fused.py -q -x 2>&1 | tail -3
