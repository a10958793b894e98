# CSR SpMV row pipelining (FITSNE_CSR_PIPE) A/B on C4 (10M random graph) + C3-CSR, one ncu --set full capture of k_attract at C4
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x -k "not c3" > gpurun_out/pytest_csrpipe.log 2>&1
for r in 1 2; do
  for v in libfitsne_b200_nopipe.so libfitsne_b200.so; do
    FITSNE_LIB=$v python bench.py --no-cpu-baseline --workload c4 > gpurun_out/abc${r}_$v.log 2>&1
  done
done
ncu --kernel-name regex:k_attract --launch-skip 3 --launch-count 1 --set full --import-source on --clock-control none \
  -f -o gpurun_out/c4_attract_full python bench.py --no-cpu-baseline --workload c4 --steps 2 --warmup 3 \
  > gpurun_out/ncu_c4.log 2>&1
