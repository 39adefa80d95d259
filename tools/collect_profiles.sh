#!/bin/bash
# Run on the GPU box:  tools/collect_profiles.sh <tag> [config]
# 1) plain bench run (must exit 0), 2) launch list with gpu__time_duration
# (serialised, cold cache), 3) --set full captures of the steady-state step
# kernels.  Outputs land in gpurun_out/; tools/summarize_profiles.py turns them
# into profiles/<tag>_*.
set -e
TAG=${1:-r01}
CFG=${2:-1}
if [ "$CFG" = "1" ]; then
  CMD="python bench.py --steps 100 --warmup 400 --no-cpu --no-e2e --instrument-steps 10"
  SKIP=1000; COUNT=2200
else
  CMD="python bench.py --config $CFG --steps 20 --warmup 200 --no-cpu --no-e2e --instrument-steps 5"
  SKIP=450; COUNT=900
fi
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none -c $COUNT --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_deliver|k_plan|k_stage" \
    -s $SKIP -c 3 -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
