# full GPU suite on the new schedule, then C3 grid sweep and the other workloads
set -x
python -m pytest tests -m gpu -q -x > gpurun_out/h_pytest_gpu.log 2>&1
tail -3 gpurun_out/h_pytest_gpu.log
B="python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz"
for c in 0 100 108 116 124; do
  $B --tiled-ctas $c > gpurun_out/h_ctas$c.log 2>&1
done
$B --side-gather 0 > gpurun_out/h_sg0.log 2>&1
python bench.py --no-cpu-baseline --shuffle > gpurun_out/h_shuffle.log 2>&1
python bench.py --no-cpu-baseline --workload c5 > gpurun_out/h_c5.log 2>&1
python bench.py --no-cpu-baseline --workload c4 > gpurun_out/h_c4.log 2>&1
