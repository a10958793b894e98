# SpMV grid scan with the vector-layout kernel
set -x
B="python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz"
for c in 112 120 124 128 132 136 148; do
  $B --tiled-ctas $c > gpurun_out/l_ctas$c.log 2>&1
done
python tools/benchline.py gpurun_out/l_ctas*.log
