# band-reduce crowding threshold: bench step and full run
set -x
B="python bench.py --no-cpu-baseline --inputs-cache /tmp/c3_inputs.npz --full-run"
$B > gpurun_out/o_c4.log 2>&1
for v in c8 c16 c32; do
  FITSNE_LIB=libfitsne_b200_$v.so $B > gpurun_out/o_$v.log 2>&1
done
python tools/benchline.py gpurun_out/o_*.log
for f in gpurun_out/o_*.log; do tail -1 $f | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('$f', d['full_run']['seconds'], d['stages']['spread']['ms'])"; done
