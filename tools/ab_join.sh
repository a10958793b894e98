# joining SpMV launch behind the repulsion chain + LPT-ordered units + streaming combine: tests, then SpMV grid A/B
set -x
python -m pytest tests/test_gpu_tiled.py tests/test_gpu_parity.py tests/test_gpu_fullrun.py tests/test_gpu_parallel.py -m gpu -x -q > gpurun_out/j_pytest.log 2>&1
tail -3 gpurun_out/j_pytest.log
B="python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz"
export FITSNE_LIB=libfitsne_b200_t.so
for c in 136 128 120 112 104; do
  $B --tiled-ctas $c > gpurun_out/j_ctas$c.log 2>&1
  grep "busy time" gpurun_out/j_ctas$c.log | tail -1
done
$B --tiled-ctas 136 --spmv-join 0 > gpurun_out/j_ctas136_nojoin.log 2>&1
$B --tiled-ctas 148 > gpurun_out/j_ctas148.log 2>&1
python tools/timeline.py --inputs-cache /tmp/c3_inputs.npz --tiled-ctas 120 > gpurun_out/j_timeline120.json 2> gpurun_out/j_timeline120.err
python tools/timeline.py --inputs-cache /tmp/c3_inputs.npz --tiled-ctas 104 > gpurun_out/j_timeline104.json 2> gpurun_out/j_timeline104.err
