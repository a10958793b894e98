# fused-iteration wall time against the SpMV grid (light chain: a run's 50-interval grid)
set -x
T="python tools/timeline_iterate.py --inputs-cache /tmp/c3_inputs.npz --schedule --at 400"
for c in 120 128 132 136 140; do $T --tiled-ctas $c > gpurun_out/s_t_$c.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/s_t_$c.json')); print($c, d['wall_us_per_iteration'])"; done
