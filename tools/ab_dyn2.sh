# dynamic unit schedule (cost-sized units), bank-ordered rows, F_rep gathered beside the SpMV: tests, then A/B
set -x
python -m pytest tests/test_gpu_tiled.py tests/test_gpu_parity.py tests/test_gpu_spread.py -m gpu -x -q > gpurun_out/d_pytest.log 2>&1
tail -3 gpurun_out/d_pytest.log
B="python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz"
for v in t t_nb t_nd t_h50; do
  FITSNE_LIB=libfitsne_b200_$v.so $B > gpurun_out/d_$v.log 2>&1
  grep "busy time" gpurun_out/d_$v.log | tail -1
done
FITSNE_LIB=libfitsne_b200_t.so $B --side-gather 0 > gpurun_out/d_t_sg0.log 2>&1
for c in 120 124 128 132; do
  FITSNE_LIB=libfitsne_b200_t.so $B --tiled-ctas $c > gpurun_out/d_t_ctas$c.log 2>&1
done
python tools/timeline.py --inputs-cache /tmp/c3_inputs.npz > gpurun_out/d_timeline.json 2> gpurun_out/d_timeline.err
python tools/timeline.py --inputs-cache /tmp/c3_inputs.npz --tiled-ctas 128 > gpurun_out/d_timeline128.json 2> gpurun_out/d_timeline128.err
python -m pytest tests/test_gpu_scale.py -m gpu -x -q > gpurun_out/d_pytest_scale.log 2>&1
tail -3 gpurun_out/d_pytest_scale.log
