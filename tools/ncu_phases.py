"""Per-phase instruction / stall-sample totals of k_stage from an ncu source
page (csv from `ncu -i X --page source --csv --print-source cuda,sass`).
Phases are delimited by the `// ---- N` markers in sim_kernels.cu."""
import csv
import re
import sys

SRC = "paper_1803_08833_b200/csrc/sim_kernels.cu"
lines = open(SRC).read().splitlines()
marks = []
for i, l in enumerate(lines, 1):
    m = re.match(r"\s*// ---- (\w+) (\w+)", l)
    if m:
        marks.append((i, f"{m.group(1)} {m.group(2)}"))
    if "// spike counter: one atomic per block" in l:
        marks.append((i, "end"))
funcs = {}
for i, l in enumerate(lines, 1):
    m = re.match(r"__device__ .*?(\w+)\(", l)
    if m:
        funcs[i] = m.group(1)


def phase(fname, ln):
    if fname != "sim_kernels.cu":
        return "lib:" + fname
    best = None
    for i, name in marks:
        if ln >= i:
            best = name
    fbest = None
    for i, name in funcs.items():
        if ln >= i and (fbest is None or i > fbest[0]):
            fbest = (i, name)
    if fbest and (not marks or ln < marks[0][0]):
        return "fn:" + fbest[1]
    return best or "setup"


rows = list(csv.reader(open(sys.argv[1])))
fname, agg, ts, ti = "", {}, 0, 0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 7 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            ln, s, i = int(r[0]), int(r[4]), int(r[7]) if r[7].isdigit() else 0
        except ValueError:
            continue
        a = agg.setdefault(phase(fname, ln), [0, 0])
        a[0] += s
        a[1] += i
        ts += s
        ti += i
for p, (s, i) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{p:28s} samples {100 * s / ts:5.1f}%  inst {i / 1e6:6.2f}M {100 * i / ti:5.1f}%")
print(f"total inst {ti / 1e6:.2f}M")
