# whole-slab split (WSLAB) and dynamic unit schedule (DYN) of the tiled SpMV: correctness, then A/B with per-CTA busy times
set -x
python -m pytest tests/test_gpu_tiled.py -m gpu -x -q > gpurun_out/w_pytest_tiled.log 2>&1
tail -3 gpurun_out/w_pytest_tiled.log
for v in libfitsne_b200_w0d0t.so libfitsne_b200_w1d1t.so libfitsne_b200_w1d0t.so libfitsne_b200_w0d1t.so libfitsne_b200.so; do
  FITSNE_LIB=$v python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz > gpurun_out/w_$v.log 2>&1
  grep "busy time" gpurun_out/w_$v.log | tail -1
  tail -1 gpurun_out/w_$v.log | cut -c1-150
done
python -m pytest tests/test_gpu_scale.py -m gpu -x -q > gpurun_out/w_pytest_scale.log 2>&1
tail -3 gpurun_out/w_pytest_scale.log
