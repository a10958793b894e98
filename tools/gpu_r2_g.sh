# Round-2 re-entry: smoke, bench, timeline, ncu --set full of one whole step's kernels, GPU suite
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1
python bench.py --inputs-cache /tmp/c3_inputs.npz > gpurun_out/g_bench.log 2>&1
python tools/timeline.py --inputs-cache /tmp/c3_inputs.npz > gpurun_out/g_timeline.json 2> gpurun_out/g_timeline.err
ncu --kernel-name regex:"k_band|k_rows|k_cols|k_spec|k_combine|k_bbox|k_attract_tiled" --launch-skip 45 --launch-count 9 \
    --set full --import-source on --clock-control none -f -o gpurun_out/g_step_full \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz > gpurun_out/g_ncu_full.log 2>&1
python -m pytest tests -m gpu -q -x > gpurun_out/g_pytest_gpu.log 2>&1
tail -3 gpurun_out/g_pytest_gpu.log
