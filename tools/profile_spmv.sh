#!/bin/bash
# full ncu capture of the fused SpMV (k_attract) in the C3 bench
TAG=${1:-spmv}
ARGS="--steps 2 --warmup 1 --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_attract" -s 3 -c 1 \
    -o gpurun_out/prof_$TAG python bench.py $ARGS > gpurun_out/ncu_$TAG.log 2>&1
echo done
