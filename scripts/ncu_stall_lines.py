"""Per-source-line warp-stall breakdown of one kernel from an ncu --set full report (imported with -lineinfo):
python scripts/ncu_stall_lines.py REP.ncu-rep [top_n]  ->  the hottest source lines with their top stall reasons."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
fname, hdr, agg = None, None, {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].isdigit():
        continue
    key = (fname, int(r[0]))
    d = agg.setdefault(key, {"src": r[1].strip()[:90], "all": 0.0, "stall": {}})
    d["all"] += float(r[4] or 0)
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            d["stall"][h[6:]] = d["stall"].get(h[6:], 0.0) + float(r[i] or 0)
tot = sum(d["all"] for d in agg.values()) or 1.0
print(f"# {rep}: {int(tot)} warp-stall samples; hottest source lines (share of samples, top reasons)")
for (f, ln), d in sorted(agg.items(), key=lambda x: -x[1]["all"])[:top]:
    st = sorted(d["stall"].items(), key=lambda x: -x[1])[:3]
    s = ", ".join(f"{k} {100 * v / max(d['all'], 1):.0f}%" for k, v in st)
    print(f"{100 * d['all'] / tot:5.1f}%  {f}:{ln:<5d} {d['src']:<90s} [{s}]")
