# A/B of tiled-SpMV variants on the C3 bench (one GPU call); results in gpurun_out/ab_*.log
set -x
python -m pytest tests -m gpu -q -k "relabel or native_nccl or tiled or parallel" > gpurun_out/pytest_ab.log 2>&1
for r in 0 1; do
  python bench.py --no-cpu-baseline --relabel $r > gpurun_out/ab_default_relabel$r.log 2>&1
done
python bench.py --no-cpu-baseline --relabel 0 --bank-order 2 > gpurun_out/ab_default_bank2.log 2>&1
FITSNE_LIB=libfitsne_b200_hoist.so python bench.py --no-cpu-baseline --relabel 0 > gpurun_out/ab_hoist_relabel0.log 2>&1
