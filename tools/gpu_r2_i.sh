# new defaults (120 CTAs, beta 1.0 / snap 1.5 cuts, polled bbox): tests, bench, timeline
set -x
python -m pytest tests/test_gpu_tiled.py tests/test_gpu_parity.py tests/test_gpu_spread.py tests/test_knn_approx.py tests/test_gpu_parallel.py -m gpu -x -q > gpurun_out/i_pytest.log 2>&1
tail -3 gpurun_out/i_pytest.log
python bench.py --inputs-cache /tmp/c3_inputs.npz > gpurun_out/i_bench.log 2>&1
tail -1 gpurun_out/i_bench.log | cut -c1-200
python tools/timeline.py --inputs-cache /tmp/c3_inputs.npz > gpurun_out/i_timeline.json 2> gpurun_out/i_timeline.err
python bench.py --no-cpu-baseline --shuffle > gpurun_out/i_shuffle.log 2>&1
python bench.py --no-cpu-baseline --workload c5 > gpurun_out/i_c5.log 2>&1
python tools/timeline.py --workload c5 > gpurun_out/i_timeline_c5.json 2> gpurun_out/i_timeline_c5.err
