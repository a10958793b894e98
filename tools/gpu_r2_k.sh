# A/B of the default build against libfitsne_b200_head.so (the previous commit's tiled.cu) and
# libfitsne_b200_x0.so (this tree without the cross-tile prefetch) on the same box
set -x
python -m pytest tests/test_gpu_tiled.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/k_pytest.log 2>&1
tail -3 gpurun_out/k_pytest.log
B="python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz"
for r in 1 2; do
FITSNE_LIB=libfitsne_b200_head.so $B > gpurun_out/k_head$r.log 2>&1
$B > gpurun_out/k_new$r.log 2>&1

done
python bench.py --no-cpu-baseline --workload c5 > gpurun_out/k_c5.log 2>&1
python tools/benchline.py gpurun_out/k_head?.log gpurun_out/k_new?.log gpurun_out/k_c5.log
