"""profiles/<tag>_kernels.md and profiles/ncu_summary.json entries from the
captures of tools/collect_r02.sh (gpurun_out/<tag>_launches.csv, _full, _b)."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

tag, key = sys.argv[1], sys.argv[2]                # e.g. r02_c1 config1
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src, dst = os.path.join(root, "gpurun_out"), os.path.join(root, "profiles")
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "smsp__inst_executed.sum", "sm__warps_active.avg.per_cycle_active",
     "smsp__average_warp_latency_per_inst_issued.ratio", "sm__cycles_active.avg",
     "sm__cycles_elapsed.avg", "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "lts__t_sectors_srcunit_tex_op_atom.sum", "lts__t_sector_hit_rate.pct",
     "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
     "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1,
         "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3, "second": 1e6}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for k, v, un in zip(h, r, u):
            if k in M:
                x = float(v.replace(",", "")) if v not in ("", "n/a") else None
                if x is not None and un in SCALE:
                    x *= SCALE[un]
                d[k] = x
        d["kernel"] = r[h.index("Kernel Name")].replace("<unnamed>::", "").replace("void ", "").split("(")[0].split("<")[0]
        res.append(d)
    return res


lines = [f"# {tag}: ncu, steady-state step kernels ({key})\n",
         "`ncu --set full --clock-control none` of two eager steps after warm-up "
         "(tools/prof_steps.py); replay (b) = k_deliver with k_stage's tail delivery off "
         "(every arrival deposited by k_deliver).  Bytes in B, times in us.\n"]
summ = {}
for suffix, label in (("_full", "steady state"), ("_b", "replay (b)")):
    rep = os.path.join(src, f"{tag}{suffix}.ncu-rep")
    if not os.path.exists(rep):
        continue
    ks = raw(rep)
    lines.append(f"\n## {label}\n\n| kernel | " + " | ".join(m.split("__")[1] for m in M) + " |\n")
    lines.append("|---" * (len(M) + 1) + "|\n")
    for d in ks:
        lines.append(f"| {d['kernel']} | " + " | ".join(
            "" if d.get(m) is None else f"{d[m]:.4g}" for m in M) + " |\n")
    for d in ks:                                   # last launch of each kernel
        name = d["kernel"] + ("_b" if suffix == "_b" else "")
        summ[name] = dict(dram_bytes_per_launch=(d["dram__bytes_read.sum"] or 0)
                          + (d["dram__bytes_write.sum"] or 0),
                          warp_instructions=d["smsp__inst_executed.sum"],
                          ipc_per_sm=(d["smsp__inst_executed.sum"] or 0)
                          / max(1.0, 148 * (d["sm__cycles_active.avg"] or 1)),
                          warps_active_per_sm=d["sm__warps_active.avg.per_cycle_active"],
                          duration_us_ncu=d["gpu__time_duration.sum"],
                          source=f"profiles/{tag}_kernels.md")
lc = os.path.join(src, f"{tag}_launches.csv")
if os.path.exists(lc):
    rows = [r for r in csv.reader(open(lc)) if len(r) > 5]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        k = r[ki].replace("<unnamed>::", "").replace("void ", "").split("(")[0]
        if k.startswith("k_"):
            k = k.split("<")[0]
        agg[k][0] += 1
        agg[k][1] += float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
    step = {k: v for k, v in agg.items() if k in ("k_deliver", "k_route", "k_bin", "k_plan", "k_stage", "k_xingest")}
    tot = sum(v[1] for v in step.values()) or 1
    lines.append("\n## launch list (bench command `--steps 20 --warmup 30`, from t = 0: onset "
                 "steps included; serialised, cold cache: compare shares)\n\n"
                 "| kernel | launches | mean us | share of step kernels |\n|---|---|---|---|\n")
    for k, (n, s) in sorted(agg.items(), key=lambda x: -x[1][1]):
        sh = f"{s / tot:.3f}" if k in step else ""
        lines.append(f"| {k} | {n} | {s / n:.1f} | {sh} |\n")
open(os.path.join(dst, f"{tag}_kernels.md"), "w").writelines(lines)
path = os.path.join(dst, "ncu_summary.json")
allj = json.load(open(path)) if os.path.exists(path) else {}
allj[key] = summ
json.dump(allj, open(path, "w"), indent=1)
print("wrote", tag, list(summ))
