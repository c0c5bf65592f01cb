"""Print the key fields of bench.py JSON lines (files given on the command line)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:   # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    r = d.get("roofline", {})
    e = d.get("e2e", {})
    print(f"{f}: {d.get('config', {}).get('workload')} value={d['value']:.3e} ms/step={d['ms_per_step']:.2f} "
          f"us/iter={r.get('us_per_iter')} bound={r.get('bound')} frac={r.get('frac')} "
          f"e2e={e.get('value') or 0:.3e} ({e.get('ms_per_step')} ms) clocks={d.get('clocks')}")
