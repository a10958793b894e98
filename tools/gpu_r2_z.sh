# host-buffer (e2e) schedules re-measured with the round's final kernels
set -x
B="python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz"
for r in 1 2; do for h in 0 1 2; do $B --host-schedule $h > gpurun_out/z_h${h}_$r.log 2>&1; done; done
python tools/benchline.py gpurun_out/z_h*.log
