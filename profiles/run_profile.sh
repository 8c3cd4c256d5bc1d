#!/bin/bash
# Reproduces the profiles committed under profiles/ (run under gpurun, 1 GPU).
#   1) launch list of the bench command (cold-cache, serialised; compare shares)
#   2) one `ncu --set full` capture of the hot kernel k_phimv_block
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_phimv_block -s 1 -c 1 \
    -o gpurun_out/prof_phimv $CMD > gpurun_out/ncu_full.log 2>&1
