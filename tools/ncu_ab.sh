#!/bin/bash
# full ncu captures (with source) of k_attract_tiled for library variants: tools/ncu_ab.sh old new ...
# ("new" = the default libfitsne_b200.so)
mkdir -p gpurun_out
for v in "$@"; do
  lib=libfitsne_b200_$v.so; [ "$v" = new ] && lib=libfitsne_b200.so
  FITSNE_LIB=$lib ncu --set full --clock-control none --import-source on -k regex:k_attract_tiled -s 1 -c 1 \
    -o gpurun_out/tiled_$v python tools/tiled_probe.py --ncu 2048,10240,148 > gpurun_out/ncu_$v.log 2>&1
  echo "$v rc=$?"
done
