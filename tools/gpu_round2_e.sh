set -x
python tools/sanitize_run.py > gpurun_out/sanitize_plain.log 2>&1
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t --error-exitcode 1 python tools/sanitize_run.py > gpurun_out/sanitizer_$t.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer_$t.log
done
python -m pytest tests -m gpu -q -k "native_nccl or parallel" > gpurun_out/pytest_nccl.log 2>&1
python bench.py --workload c4 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
python bench.py --workload c5 > gpurun_out/bench_c5.log 2>&1
