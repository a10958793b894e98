# A/B of tiled-SpMV build variants (FITSNE_LIB) on the C3 bench
set -x
python -m pytest tests -m gpu -q -k "tiled" > gpurun_out/pytest_ab2.log 2>&1
for v in libfitsne_b200.so libfitsne_b200_nopf.so libfitsne_b200_u8t768.so; do
  FITSNE_LIB=$v python bench.py --no-cpu-baseline > gpurun_out/ab2_$v.log 2>&1
done
