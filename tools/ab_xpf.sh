# tiled SpMV: cross-tile first-batch prefetch (FITSNE_TILED_XPF) and shared-memory CAS flush of cut slabs (FITSNE_TILED_SCUT)
set -x
for v in libfitsne_b200.so libfitsne_b200_scut.so; do
  FITSNE_LIB=$v timeout 900 python -m pytest tests/test_gpu_tiled.py -m gpu -q -x > gpurun_out/pytest_xpf_$v.log 2>&1
done
for r in 1 2; do
  for v in libfitsne_b200_noxpf.so libfitsne_b200.so libfitsne_b200_scut.so; do
    FITSNE_LIB=$v python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz > gpurun_out/abx${r}_$v.log 2>&1
  done
done
for v in libfitsne_b200_noxpf.so libfitsne_b200.so libfitsne_b200_scut.so; do
  FITSNE_LIB=$v python bench.py --no-cpu-baseline --workload c5 > gpurun_out/abx_c5_$v.log 2>&1
done
