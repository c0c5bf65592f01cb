#!/bin/bash
# k_batch_chain: parity subset + C5/C2 bench lines (new kernel and the previous one for A/B)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "cluster or c2 or c5 or precomputed or chain or freeze" > gpurun_out/chain_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/chain_tests.log
tail -3 gpurun_out/chain_tests.log
for w in C5 C2; do
  timeout 600 python bench.py --workload $w --steps 3 --warmup 1 --no-cpu --no-e2e > gpurun_out/chain_$w.json 2> gpurun_out/chain_$w.err
  COT_BATCH_CHAIN=0 timeout 600 python bench.py --workload $w --steps 3 --warmup 1 --no-cpu --no-e2e > gpurun_out/old_$w.json 2> gpurun_out/old_$w.err
done
python - <<'PY'
import json
for f in ["chain_C5", "old_C5", "chain_C2", "old_C2"]:
    try:
        d = json.load(open(f"gpurun_out/{f}.json"))
        r = d["roofline"]
        print(f, f"{d['value']:.3e}", d["ms_per_step"], "frac", round(r["frac"], 3), "us/iter", round(r["us_per_iter"], 3), d["clocks"]["sm_mhz"])
    except Exception as e:
        print(f, "ERR", e, open(f"gpurun_out/{f}.err").read()[-800:])
PY
