set -x
python -m pytest tests/test_gpu_spread.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/n_pytest.log 2>&1
tail -3 gpurun_out/n_pytest.log
T="python tools/timeline_iterate.py --inputs-cache /tmp/c3_inputs.npz"
$T --at 10 > gpurun_out/n_t_collapsed.json 2>/dev/null
$T --at 10 --overlap 0 > gpurun_out/n_t_collapsed_serial.json 2>/dev/null
python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz --full-run > gpurun_out/n_bench_fullrun.log 2>&1
python tools/benchline.py gpurun_out/n_bench_fullrun.log
