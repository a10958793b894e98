# kernel spectrum ahead of the spread (FITSNE_OPT_SPEC_AHEAD): tests, bench A/B, timelines
set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_spread.py tests/test_gpu_fullrun.py tests/test_gpu_reference_suite.py -m gpu -x -q > gpurun_out/v_pytest.log 2>&1
tail -3 gpurun_out/v_pytest.log
B="python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz"
for r in 1 2; do
$B > gpurun_out/v_on$r.log 2>&1
$B --spec-ahead 0 > gpurun_out/v_off$r.log 2>&1
done
python tools/benchline.py gpurun_out/v_on?.log gpurun_out/v_off?.log
python tools/timeline.py --inputs-cache /tmp/c3_inputs.npz > gpurun_out/v_timeline.json 2>/dev/null
python tools/timeline_iterate.py --inputs-cache /tmp/c3_inputs.npz --schedule --at 400 > gpurun_out/v_titer.json 2>/dev/null
