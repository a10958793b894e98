for c in 1 2 4; do
  python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz --fft-cols $c --breakdown > gpurun_out/ab_fftcols_$c.log 2>&1
done
