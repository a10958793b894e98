# SpMV persistent-grid sweep on the C3 bench (the repulsion chain gets the other SMs)
for c in 0 112 120 124 128 132; do
  python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz --tiled-ctas $c > gpurun_out/ab_ctas_$c.log 2>&1
done
