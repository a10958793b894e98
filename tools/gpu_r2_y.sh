# dynamic-schedule knobs (static head share, tail unit size) with the vector-layout kernel
set -x
B="python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz"
for r in 1 2 3; do
$B > gpurun_out/y_default$r.log 2>&1
for v in h85 h92 h85u12; do FITSNE_LIB=libfitsne_b200_$v.so $B > gpurun_out/y_$v$r.log 2>&1; done
done
python tools/benchline.py gpurun_out/y_default?.log gpurun_out/y_h85?.log gpurun_out/y_h92?.log gpurun_out/y_h85u12?.log
