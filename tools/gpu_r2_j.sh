# vector slot layout / packed warp descriptors: tests, A/B against HEAD's tiled.cu on the same box
set -x
python -m pytest tests/test_gpu_tiled.py tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -x -q > gpurun_out/j_pytest.log 2>&1
tail -3 gpurun_out/j_pytest.log
B="python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz"
FITSNE_LIB=libfitsne_b200_head.so $B > gpurun_out/j_head.log 2>&1
$B > gpurun_out/j_new.log 2>&1
FITSNE_LIB=libfitsne_b200_v0.so $B > gpurun_out/j_v0.log 2>&1
FITSNE_LIB=libfitsne_b200_head.so $B > gpurun_out/j_head2.log 2>&1
$B > gpurun_out/j_new2.log 2>&1
FITSNE_LIB=libfitsne_b200_v0.so $B > gpurun_out/j_v02.log 2>&1
python bench.py --no-cpu-baseline --workload c5 > gpurun_out/j_c5.log 2>&1
python tools/benchline.py gpurun_out/j_head.log gpurun_out/j_new.log gpurun_out/j_v0.log gpurun_out/j_head2.log gpurun_out/j_new2.log gpurun_out/j_v02.log gpurun_out/j_c5.log
