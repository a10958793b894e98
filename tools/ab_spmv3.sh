# debug-bounds test run + tiled-SpMV pipeline variants (FITSNE_LIB) on the C3 bench
set -x
FITSNE_LIB=libfitsne_b200_debug.so timeout 1500 python -m pytest tests -m gpu -q -k "not scale" > gpurun_out/pytest_debug_bounds.log 2>&1
for v in libfitsne_b200.so libfitsne_b200_fast.so libfitsne_b200_d3.so libfitsne_b200_d3t768.so libfitsne_b200_d3t512.so libfitsne_b200_u8d3t512.so; do
  FITSNE_LIB=$v python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz > gpurun_out/ab3_$v.log 2>&1
done
