#!/bin/bash
# ncu evidence for the C3 bench (run under gpurun, 1 GPU).
#  1. plain run (must exit 0 before ncu is used)
#  2. launch list of the library's kernels (serialised, cold-cache durations)
#  3. one --set full capture of each kernel of one gradient evaluation
set -e
TAG=${1:-r06}
ARGS="--steps 2 --warmup 1 --no-cpu-baseline"
mkdir -p gpurun_out
python bench.py $ARGS > gpurun_out/plain_$TAG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py $ARGS > gpurun_out/ncu_list_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_attract|k_spread|k_band|k_cols|k_spec_cols|k_rows_forward|k_rows_inverse|k_combine|k_bbox|k_box|k_tiled" \
    -s 14 -c 16 -o gpurun_out/prof_$TAG python bench.py $ARGS > gpurun_out/ncu_full_$TAG.log 2>&1
echo done
