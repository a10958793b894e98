# tiled SpMV: shared-memory CAS flush of cut slabs (FITSNE_TILED_SCUT) vs default; two tile shapes
set -x
for r in 1 2; do
  for v in libfitsne_b200.so libfitsne_b200_scut.so; do
    FITSNE_LIB=$v python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz > gpurun_out/abs${r}_$v.log 2>&1
    FITSNE_LIB=$v python bench.py --no-cpu-baseline --workload c5 > gpurun_out/abs${r}_c5_$v.log 2>&1
  done
done
for t in 2048x8192 4096x6144; do
  python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz --tile $t > gpurun_out/abs_tile_$t.log 2>&1
done
