# ring depth x tile shape (the consumers stall at tile starts waiting for the next Y chunk)
python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz > gpurun_out/ab_st2_3072x8192.log 2>&1
python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz --tile 2048x6144 > gpurun_out/ab_st2_2048x6144.log 2>&1
for t in 2048x6144 2560x6144 1536x8192 2048x7168; do
  FITSNE_LIB=libfitsne_b200_s3.so python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz --tile $t > gpurun_out/ab_st3_$t.log 2>&1
done
