# cost-balanced warp cuts inside a tile (beta = slab-boundary cost, snap = move cuts onto slab boundaries)
set -x
python -m pytest tests/test_gpu_tiled.py tests/test_knn_approx.py -m gpu -x -q > gpurun_out/c_pytest.log 2>&1
tail -3 gpurun_out/c_pytest.log
B="python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz"
for v in c00 b15s10 b15s0 b25s10 b10s15 b20s20; do
  FITSNE_LIB=libfitsne_b200_$v.so $B > gpurun_out/c_$v.log 2>&1
  grep "busy time" gpurun_out/c_$v.log | tail -1
done
for m in 1 4; do
  FITSNE_LIB=libfitsne_b200_b15s10.so $B --overlap-mode $m --tiled-ctas 112 > gpurun_out/c_ov${m}_112.log 2>&1
  FITSNE_LIB=libfitsne_b200_b15s10.so $B --overlap-mode $m --tiled-ctas 136 > gpurun_out/c_ov${m}_136.log 2>&1
done
