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
config = int(sys.argv[2]) if len(sys.argv) > 2 else 1
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = os.path.join(root, "gpurun_out")
dst = os.path.join(root, "profiles")
os.makedirs(dst, exist_ok=True)

# --- launch list: share of step time per kernel (steady state = last 400 launches of step kernels)
have_launches = os.path.exists(os.path.join(src, f"{tag}_launches.csv"))
rows = [r for r in csv.reader(open(os.path.join(src, f"{tag}_launches.csv"))) if len(r) > 5] \
    if have_launches else [["Kernel Name", "Metric Value", "Metric Unit", "", "", ""]]
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
with open(os.path.join(dst, f"{tag}_launches.md") if have_launches else os.devnull, "w") as fh:
    fh.write(f"# {tag}: ncu launch list (gpu__time_duration, --clock-control none)\n\n")
    fh.write(("Command: `python bench.py --steps 100 --warmup 400 --no-cpu --no-e2e "
              "--instrument-steps 10`" if config == 1 else
              f"Command: `python bench.py --config {config} --steps 20 --warmup 200 --no-cpu "
              "--no-e2e --instrument-steps 5`") +
             " under `ncu --metrics gpu__time_duration.sum`.\n"
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
        "lts__t_bytes.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex_op_atom.sum",
        "lts__t_sectors_srcunit_tex_op_write.sum", "lts__t_sectors_srcunit_tex_op_read.sum"]
units = raw[1]
summary = {}
with open(os.path.join(dst, f"{tag}_kernels.md"), "w") as fh:
    fh.write(f"# {tag}: ncu --set full, steady-state step kernels, BASELINE config {config}\n\n")
    for r in raw[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        d = {}
        for k in keys:
            if k in h:
                d[k] = (r[h.index(k)], units[h.index(k)])
        fh.write(f"## {name}\n\n| metric | value | unit |\n|---|---|---|\n")
        for k, (v, u) in d.items():
            fh.write(f"| {k} | {v} | {u} |\n")
        st = sorted(((h[i].replace("smsp__average_warps_issue_stalled_", "")
                      .replace("_per_issue_active.ratio", ""), float(r[i] or 0))
                     for i in range(len(h)) if h[i].startswith("smsp__average_warps_issue_stalled_")
                     and h[i].endswith("_per_issue_active.ratio")), key=lambda x: -x[1])[:6]
        fh.write("\nwarp stall cycles per issued instruction: "
                 + ", ".join(f"{k} {v:.2f}" for k, v in st) + "\n\n")

        def num(k):
            v, u = d.get(k, ("0", ""))
            x = float(v.replace(",", ""))
            return x * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1}.get(u, 1)
        summary[name.split("<")[0]] = {
            "dram_bytes_per_launch": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
            "warp_instructions": num("smsp__inst_executed.sum"),
            "ipc_per_sm": (num("smsp__inst_executed.sum") / max(1.0, num("sm__cycles_active.avg"))
                           / 148.0),
            "warps_active_per_sm": num("sm__warps_active.avg.per_cycle_active"),
            "duration_us_ncu": float(d["gpu__time_duration.sum"][0].replace(",", "")) *
            {"nsecond": 1e-3, "ns": 1e-3, "msecond": 1e3, "ms": 1e3}.get(
                d["gpu__time_duration.sum"][1], 1.0),
            "source": f"profiles/{tag}_kernels.md"}
path = os.path.join(dst, "ncu_summary.json")
allsum = json.load(open(path)) if os.path.exists(path) else {}
allsum = {k: v for k, v in allsum.items() if k.startswith("config")}   # older flat layout
allsum[f"config{config}"] = summary
json.dump(allsum, open(path, "w"), indent=1)
if have_launches:
    print(open(os.path.join(dst, f"{tag}_launches.md")).read())
print(json.dumps(summary, indent=1))
