# C4 CSR SpMV: L2 set-aside for the evict_last Y gathers (FITSNE_OPT_L2_PERSIST)
set -x
python -c "import torch; p=torch.cuda.get_device_properties(0); print('persist_max', p.persisting_l2_cache_max_size, 'l2', p.L2_cache_size)" > gpurun_out/l2_props.log 2>&1
for mb in 0 96 0 96 48; do
  python bench.py --no-cpu-baseline --workload c4 --l2-persist $mb > gpurun_out/abl_${mb}_$RANDOM.log 2>&1
done
