#!/bin/bash
# Capture steady-state launches of the step kernels with ncu (run on the GPU box).
# usage: tools/profile_kernels.sh <tag> [kernel-regex]
set -e
TAG=${1:-cur}
RE=${2:-"k_stage|k_update|k_deliver"}
CMD="python bench.py --steps 100 --warmup 400 --no-cpu --no-e2e --instrument-steps 10"
$CMD > gpurun_out/plain_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"$RE" -s ${SKIP:-450} -c ${COUNT:-1} \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1 || tail -5 gpurun_out/ncu_$TAG.log
