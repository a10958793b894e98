set -x
T="python tools/timeline_iterate.py --inputs-cache /tmp/c3_inputs.npz --schedule"
for a in 150 400 650 850; do $T --at $a > gpurun_out/q_t_$a.json 2>/dev/null; done
