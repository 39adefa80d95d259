"""Summarise an ncu report: per kernel duration, SM activity, CPI, top lines,
and per-stage instruction counts for k_stage (stage markers '// ---- ')."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
src_file = "/root/repo/paper_1803_08833_b200/csrc/sim_kernels.cu"


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
h = raw[0]
want = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
        "smsp__inst_executed.sum", "smsp__average_warp_latency_per_inst_issued.ratio",
        "sm__warps_active.avg.per_cycle_active", "launch__grid_size", "launch__registers_per_thread",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum"]
idx = [h.index(w) for w in want if w in h]
for r in raw[2:]:
    print({h[i]: r[i] for i in idx})
src = open(src_file).read().split("\n")
marks = [(i + 1, l.strip()[:60]) for i, l in enumerate(src) if "// ---- " in l or "__global__" in l]
txt = run("--page", "source", "--csv", "--print-source", "cuda,sass")
rows = list(csv.reader(io.StringIO(txt)))
fname = ""
func = ""
agg = {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Function Name":
        func = r[1]
        continue
    if len(r) > 7 and r[0] not in ("", "Line No") and r[2] == "-" and fname == "sim_kernels.cu":
        try:
            ln, smp, ins = int(r[0]), int(r[4]), int(r[7])
        except ValueError:
            continue
        name = "?"
        for m_ln, m_name in marks:
            if m_ln <= ln:
                name = m_name
        key = (func[:40], name)
        a = agg.setdefault(key, [0, 0])
        a[0] += smp
        a[1] += ins
for (f, n), (smp, ins) in sorted(agg.items(), key=lambda x: -x[1][0])[:30]:
    print(f"{f:40s} {n:60s} samples {smp:6d} inst {ins/1e6:7.3f}M")
