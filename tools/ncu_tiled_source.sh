# One ncu --set full capture (with source) of the tiled SpMV inside the C3 bench
# step; read it locally with: ncu -i gpurun_out/tiled_full.ncu-rep --page source --csv
ncu --kernel-name regex:k_attract_tiled --launch-skip 5 --launch-count 1 --set full \
    --import-source on --clock-control none -f -o gpurun_out/tiled_full \
    python bench.py --no-cpu-baseline --steps 3 --warmup 3 "$@" > gpurun_out/ncu_tiled_full.log 2>&1
