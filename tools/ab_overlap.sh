python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz --overlap-mode 1 > gpurun_out/ab_ov1.log 2>&1
for c in 0 140 144; do
  python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz --overlap-mode 3 --tiled-ctas $c > gpurun_out/ab_ov3_$c.log 2>&1
done
python tools/timeline.py --inputs-cache /tmp/c3_inputs.npz --overlap 3 > gpurun_out/timeline_ov3.json 2>gpurun_out/timeline_ov3.err
