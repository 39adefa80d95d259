"""Aggregate ncu source-page warp-stall samples per CUDA source line.
usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > f.csv; python tools/ncu_lines.py f.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
out = []
fname = ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 6 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            out.append((int(r[4]), int(r[7]) if r[7].isdigit() else 0, f"{fname}:{r[0]}", r[1][:100]))
        except ValueError:
            pass
tot = sum(o[0] for o in out) or 1
for s, ins, loc, src in sorted(out, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{s:7d} {100 * s / tot:5.1f}% inst={ins:9d} {loc:24s} {src}")
