set -x
python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz --relabel 2 > gpurun_out/ab_relabel2_pf.log 2>&1
python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz --relabel 0 > gpurun_out/ab_relabel0_pf.log 2>&1
python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz --full-run > gpurun_out/bench_c3_fullrun.log 2>&1
python bench.py --workload c5 --no-cpu-baseline --full-run > gpurun_out/bench_c5_fullrun.log 2>&1
