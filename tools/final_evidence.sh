# Round evidence on one B200: GPU suite, smoke, the driver's bench command,
# the ncu launch list of the same command and one --set full capture of the
# dominant kernel (read back with tools/ncu_summary.py / tools/ncu_src_wavefronts.py into profiles/).
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1
python -m pytest tests -m gpu -q > gpurun_out/ev_pytest_gpu.log 2>&1
tail -3 gpurun_out/ev_pytest_gpu.log
python bench.py > gpurun_out/ev_bench.log 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev_bench_reference.log 2>&1
ncu --nvtx --nvtx-include "bench_step/" --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/ev_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_launches.log 2>&1
# the step launches the tiled kernel twice (main grid + the joining launch): capture both, the summary picks the long one
ncu --kernel-name regex:k_attract_tiled --launch-skip 6 --launch-count 2 --set full --import-source on \
    --clock-control none -f -o gpurun_out/ev_tiled_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ev_ncu_full.log 2>&1
python tools/timeline.py > gpurun_out/ev_timeline.json 2> gpurun_out/ev_timeline.err
python bench.py --shuffle --no-cpu-baseline > gpurun_out/ev_bench_shuffle.log 2>&1
python bench.py --workload c5 --full-run > gpurun_out/ev_bench_c5.log 2>&1
python bench.py --workload c4 --no-cpu-baseline > gpurun_out/ev_bench_c4.log 2>&1
python bench.py --full-run --no-cpu-baseline > gpurun_out/ev_bench_c3_fullrun.log 2>&1
python tools/benchline.py gpurun_out/ev_bench.log gpurun_out/ev_bench_shuffle.log gpurun_out/ev_bench_c5.log gpurun_out/ev_bench_c4.log gpurun_out/ev_bench_c3_fullrun.log
