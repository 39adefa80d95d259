#!/bin/bash
# A/B of library variants on one box: tools/ab.sh "<bench args>" name1 name2 ...
# (build_variants/lib_<name>.so, built here with tools/sweep_variants.py or
# paper_1803_08833_b200.build.build(out=..., defines=...)); prints ms/step.
ARGS="$1"; shift
for v in "$@"; do
  CC_LIB_PATH=build_variants/lib_$v.so python bench.py --no-cpu --no-e2e $ARGS > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err \
    || { echo "$v FAILED"; tail -3 gpurun_out/ab_$v.err; continue; }
  python - "$v" <<'P'
import json, sys
v = sys.argv[1]
d = json.load(open(f"gpurun_out/ab_{v}.json"))
k = d["kernels"]
print(f"{v:16s} ms/step {d['ms_per_step']*1e3:8.2f} us  value {d['value']:.4e}  del {k['k_deliver']['avg_us']:.1f} "
      f"neu {k['k_neuron']['avg_us']:.1f}  (b) del {k['k_deliver_all_arrivals']['avg_us']:.1f}  grid {d.get('stage_grid',{}).get('warps')}")
P
done
