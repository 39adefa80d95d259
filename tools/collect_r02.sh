#!/bin/bash
# Run on the GPU box:  tools/collect_r02.sh <tag> <config> [regime] [grid]
# 1) launch list of the bench command (ncu gpu__time_duration, serialised),
# 2) --set full captures of two steady-state steps (all step kernels),
# 3) --set full capture of k_deliver (or k_route + k_bin) with k_stage's tail delivery off (the
#    bench's roofline replay (b)).  tools/summarize_r02.py writes profiles/.
TAG=${1:-r02}; CFG=${2:-1}; REG=${3:-calibrated}; GRID=${4:-}
N=/usr/local/cuda/bin/ncu
G=""; [ -n "$GRID" ] && G="--grid $GRID"
W=400; [ "$CFG" != "1" ] && W=200
$N --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
   python bench.py --config $CFG --regime $REG $G --steps 20 --warmup 30 --no-cpu --no-e2e --instrument-steps 5 \
   > gpurun_out/${TAG}_launches.log 2>&1; echo launches=$?
$N --set full --clock-control none --import-source on --profile-from-start off -o gpurun_out/${TAG}_full \
   python tools/prof_steps.py --config $CFG --regime $REG $G --warmup $W --steps 2 > gpurun_out/${TAG}_full.log 2>&1; echo full=$?
$N --set full --clock-control none --import-source on --profile-from-start off -k "regex:k_deliver|k_route|k_bin" -o gpurun_out/${TAG}_b \
   python tools/prof_steps.py --config $CFG --regime $REG $G --warmup $W --steps 2 --flags 4096 > gpurun_out/${TAG}_b.log 2>&1; echo b=$?
