# warp-cut cost model (beta = slab start cost in groups, snap = snap distance) with the vector-layout kernel
set -x
B="python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz"
for v in b05 b15 b20 b25; do
  FITSNE_LIB=libfitsne_b200_$v.so $B > gpurun_out/m_$v.log 2>&1
done
$B > gpurun_out/m_default.log 2>&1
python tools/benchline.py gpurun_out/m_*.log
