"""Turn gpurun_out/<tag>_* (tools/collect_profiles.sh) into committed
profiles/<tag>_launches.md, profiles/<tag>_kernels.md and profiles/ncu_summary.json."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = os.path.join(root, "gpurun_out")
dst = os.path.join(root, "profiles")
os.makedirs(dst, exist_ok=True)

# --- launch list: share of step time per kernel (steady state = last 400 launches of step kernels)
rows = [r for r in csv.reader(open(os.path.join(src, f"{tag}_launches.csv"))) if len(r) > 5]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
launches = []
for r in rows[1:]:
    v = float(r[vi].replace(",", ""))
    if r[ui] in ("nsecond", "ns"):
        v /= 1e3
    elif r[ui] in ("msecond", "ms"):
        v *= 1e3
    launches.append((r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", ""), v))
step_k = [l for l in launches if l[0].split("<")[0] in ("k_deliver", "k_plan", "k_stage", "k_update")]
tail = step_k[-400:]
agg = defaultdict(lambda: [0, 0.0])
for k, v in tail:
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(a[1] for a in agg.values())
with open(os.path.join(dst, f"{tag}_launches.md"), "w") as fh:
    fh.write(f"# {tag}: ncu launch list (gpu__time_duration, --clock-control none)\n\n")
    fh.write("Command: `python bench.py --steps 100 --warmup 400 --no-cpu --no-e2e "
             "--instrument-steps 10` under `ncu --metrics gpu__time_duration.sum`.\n"
             "Serialised, cold-cache per-launch times: compare SHARES, not absolutes.\n\n")
    fh.write(f"Total launches captured: {len(launches)}; step-kernel launches: {len(step_k)}; "
             f"summary over the last {len(tail)} step-kernel launches.\n\n")
    fh.write("| kernel | launches | mean us | share of step |\n|---|---|---|---|\n")
    for k, (n, s) in sorted(agg.items(), key=lambda x: -x[1][1]):
        fh.write(f"| {k} | {n} | {s / n:.1f} | {s / tot:.3f} |\n")
    other = defaultdict(lambda: [0, 0.0])
    for k, v in launches:
        if (k, v) not in tail:
            other[k][0] += 1
            other[k][1] += v
    fh.write("\nAll kernels over the whole run:\n\n| kernel | launches | total us |\n|---|---|---|\n")
    allk = defaultdict(lambda: [0, 0.0])
    for k, v in launches:
        allk[k][0] += 1
        allk[k][1] += v
    for k, (n, s) in sorted(allk.items(), key=lambda x: -x[1][1]):
        fh.write(f"| {k} | {n} | {s:.1f} |\n")

# --- full captures
rep = os.path.join(src, f"{tag}_full.ncu-rep")
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                                 capture_output=True, text=True).stdout)))
h = raw[0]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__cycles_active.avg", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
        "smsp__average_warp_latency_per_inst_issued.ratio", "sm__warps_active.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]
units = raw[1]
summary = {}
with open(os.path.join(dst, f"{tag}_kernels.md"), "w") as fh:
    fh.write(f"# {tag}: ncu --set full, steady-state step kernels (launch ~1350+)\n\n")
    for r in raw[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        d = {}
        for k in keys:
            if k in h:
                d[k] = (r[h.index(k)], units[h.index(k)])
        fh.write(f"## {name}\n\n| metric | value | unit |\n|---|---|---|\n")
        for k, (v, u) in d.items():
            fh.write(f"| {k} | {v} | {u} |\n")
        fh.write("\n")

        def num(k):
            v, u = d.get(k, ("0", ""))
            x = float(v.replace(",", ""))
            return x * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1}.get(u, 1)
        summary[name.split("<")[0]] = {
            "dram_bytes_per_launch": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
            "duration_us_ncu": float(d["gpu__time_duration.sum"][0].replace(",", "")) /
            (1e3 if d["gpu__time_duration.sum"][1] in ("nsecond", "ns") else 1),
            "source": f"profiles/{tag}_kernels.md"}
json.dump(summary, open(os.path.join(dst, "ncu_summary.json"), "w"), indent=1)
print(open(os.path.join(dst, f"{tag}_launches.md")).read())
print(json.dumps(summary, indent=1))
