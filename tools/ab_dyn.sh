# tiled SpMV: previous commit vs producer TileLoad prefetch vs dynamic chunk split (FITSNE_TILED_DYN)
set -x
FITSNE_LIB=libfitsne_b200_dyn.so timeout 900 python -m pytest tests/test_gpu_tiled.py tests/test_gpu_scale.py -m gpu -q -x > gpurun_out/pytest_dyn.log 2>&1
for r in 1 2; do
  for v in libfitsne_b200_prev.so libfitsne_b200.so libfitsne_b200_dyn.so; do
    FITSNE_LIB=$v python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz > gpurun_out/abd${r}_$v.log 2>&1
  done
done
FITSNE_LIB=libfitsne_b200_dyn.so python bench.py --no-cpu-baseline --shuffle > gpurun_out/abd_dyn_shuffle.log 2>&1
FITSNE_LIB=libfitsne_b200_dyn.so python bench.py --no-cpu-baseline --workload c5 > gpurun_out/abd_dyn_c5.log 2>&1
ncu --kernel-name regex:'^k_' --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/launches_c3.csv python bench.py --no-cpu-baseline --steps 3 --warmup 3 --inputs-cache /tmp/c3_inputs.npz > gpurun_out/ncu_launch.log 2>&1
