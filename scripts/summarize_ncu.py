"""Summarise gpurun_out/ ncu artefacts into profiles/ (tracked): launch shares + key metrics of the top kernel.
usage: python scripts/summarize_ncu.py <round_tag> <workload> <launches.csv> <prof.ncu-rep> [iters_in_profiled_launch]"""
import collections
import csv
import json
import os
import subprocess
import sys

tag, workload, launches, rep = sys.argv[1:5]
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 1
out_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
os.makedirs(out_dir, exist_ok=True)

rows = [r for r in csv.reader(open(launches)) if len(r) > 5]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(list)
for r in rows[1:]:
    v = float(r[vi].replace(",", ""))
    v = {"ns": v / 1e3, "us": v, "usecond": v, "ms": v * 1e3, "msecond": v * 1e3, "nsecond": v / 1e3}.get(r[ui], v)
    agg[r[ki].split("(")[0].strip()].append(v)
tot = sum(sum(v) for v in agg.values())
lines = [f"# {tag} launch list ({workload}): ncu --metrics gpu__time_duration.sum --clock-control none, one step",
         "# cold-cache, serialised per-launch times: compare SHARES, not absolutes", "kernel,launches,mean_us,total_ms,share"]
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    lines.append(f"{k},{len(v)},{sum(v)/len(v):.2f},{sum(v)/1e3:.4f},{sum(v)/tot:.4f}")
open(os.path.join(out_dir, f"{tag}_{workload}_launches.csv"), "w").write("\n".join(lines) + "\n")

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, u, v = r[0], r[1], r[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second"]
met = {}
for k in want:
    if k in h:
        met[k] = {"value": v[h.index(k)], "unit": u[h.index(k)]}
open(os.path.join(out_dir, f"{tag}_{workload}_top_kernel_metrics.json"), "w").write(json.dumps(met, indent=1) + "\n")
with open(os.path.join(out_dir, f"{tag}_{workload}_top_kernel_raw.csv"), "w") as f:
    f.write(raw)


def to_bytes(d):
    x = float(d["value"].replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(d["unit"], 1)


summ_path = os.path.join(out_dir, "ncu_summary.json")
summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
traffic = (to_bytes(met["dram__bytes_read.sum"]) + to_bytes(met["dram__bytes_write.sum"])) / iters
summ[workload] = {"round": tag, "k_rows_dram_bytes_per_launch": None, "kernel": met.get("Kernel Name", {}).get("value"),
                  "dram_bytes_per_iteration": traffic, "profiled_iterations": iters}
json.dump(summ, open(summ_path, "w"), indent=1)
print("\n".join(lines))
print(json.dumps(met, indent=1))
