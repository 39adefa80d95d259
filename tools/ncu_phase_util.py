"""Per-phase warp instructions, thread instructions (lane utilisation) and
stall samples of a kernel from an ncu source page csv
(`ncu -i X --page source --csv --print-source cuda,sass -k regex:K`).
Phases: the `// ---- N name` markers of sim_kernels.cu, device functions by name."""
import csv
import re
import sys

SRC = "paper_1803_08833_b200/csrc/sim_kernels.cu"
lines = open(SRC).read().splitlines()
marks, funcs = [], []
for i, l in enumerate(lines, 1):
    m = re.match(r"\s*// ---- (\w+) (\w+)", l)
    if m:
        marks.append((i, f"{m.group(1)} {m.group(2)}"))
    if "// spike counter: one atomic per block" in l:
        marks.append((i, "end"))
    m = re.match(r"(?:__device__|__global__|template).*?\b(\w+)\s*\(", l)
    if m and "k_stage" not in l:
        funcs.append((i, m.group(1)))
    if re.match(r"k_stage\(", l) or "k_stage(const cc_shard sh)" in l:
        funcs.append((i, "k_stage"))
funcs.sort()


def phase(fname, ln):
    if fname != "sim_kernels.cu":
        return "lib:" + fname
    f = None
    for i, name in funcs:
        if ln >= i:
            f = name
    if f == "k_stage":
        best = "k_stage:setup"
        for i, name in marks:
            if ln >= i:
                best = name
        return best
    return "fn:" + (f or "?")


rows = list(csv.reader(open(sys.argv[1])))
fname, agg = "", {}
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))
    try:
        ln = int(r[0])
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        wi = int(d.get("Instructions Executed", "0") or 0)
        ti = int(d.get("Thread Instructions Executed", "0") or 0)
    except ValueError:
        continue
    a = agg.setdefault(phase(fname, ln), [0, 0, 0])
    a[0] += s; a[1] += wi; a[2] += ti
ts = sum(a[0] for a in agg.values()) or 1
tw = sum(a[1] for a in agg.values()) or 1
for p, (s, wi, ti) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{p:26s} stall-samples {100 * s / ts:5.1f}%  warp-inst {wi / 1e6:7.2f}M {100 * wi / tw:5.1f}%"
          f"  lanes/inst {ti / max(wi, 1):5.1f}")
print(f"total warp inst {tw / 1e6:.2f}M, thread inst {sum(a[2] for a in agg.values()) / 1e6:.1f}M")
