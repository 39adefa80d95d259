#!/bin/bash
# Per-kernel mean time over steady-state steps (serialised by ncu; compare shares).
CMD="python bench.py --steps 20 --warmup 300 --no-cpu --no-e2e --instrument-steps 5"
ncu --metrics gpu__time_duration.sum --clock-control none -s 900 -c 45 --csv \
    --log-file gpurun_out/lt.csv $CMD > /dev/null 2>&1
python3 - <<'PY'
import csv
from collections import defaultdict
rows=[r for r in csv.reader(open('gpurun_out/lt.csv')) if len(r)>5]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
a=defaultdict(list)
for r in rows[1:]:
    a[r[ki].split('(')[0].replace('void ','').replace('<unnamed>::','')].append(float(r[vi].replace(',',''))/1e3)
tot=sum(sum(v)/len(v) for v in a.values())
for k,v in sorted(a.items(), key=lambda x:-sum(x[1])/len(x[1])):
    print(f"{k:20s} n={len(v):3d} mean {sum(v)/len(v):8.1f} us  share {sum(v)/len(v)/tot:.3f}")
PY
