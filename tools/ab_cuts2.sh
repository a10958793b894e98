# beta / snap scan of the cost-balanced warp cuts, then SpMV grid scan with the best so far
set -x
B="python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz"
for v in b5s15 b8s15 b10s15 b10s25 b12s20 b8s30; do
  FITSNE_LIB=libfitsne_b200_$v.so $B > gpurun_out/c2_$v.log 2>&1
  grep "busy time" gpurun_out/c2_$v.log | tail -1
done
for c in 104 112 120 128; do
  FITSNE_LIB=libfitsne_b200_b10s15.so $B --tiled-ctas $c > gpurun_out/c2_b10s15_ctas$c.log 2>&1
done
FITSNE_LIB=libfitsne_b200_b10s15.so python bench.py --no-cpu-baseline --workload c5 > gpurun_out/c2_c5.log 2>&1
FITSNE_LIB=libfitsne_b200_b10s15.so python bench.py --no-cpu-baseline --workload c5 --spmv-join 0 > gpurun_out/c2_c5_nojoin.log 2>&1
