# Round evidence on one B200: GPU suite, smoke, the driver's bench command,
# the ncu launch list of the same command and one --set full capture of the
# dominant kernel (read back with tools/ncu_summary.py into profiles/).
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1
python -m pytest tests -m gpu -q > gpurun_out/ev_pytest_gpu.log 2>&1
python bench.py > gpurun_out/ev_bench.log 2>&1
ncu --nvtx --nvtx-include "bench_step/" --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/ev_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_launches.log 2>&1
ncu --kernel-name regex:k_attract_tiled --launch-skip 5 --launch-count 1 --set full --import-source on \
    --clock-control none -f -o gpurun_out/ev_tiled_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ev_ncu_full.log 2>&1
python bench.py --shuffle --no-cpu-baseline > gpurun_out/ev_bench_shuffle.log 2>&1
python bench.py --workload c5 --full-run > gpurun_out/ev_bench_c5.log 2>&1
python bench.py --full-run --no-cpu-baseline > gpurun_out/ev_bench_c3_fullrun.log 2>&1
