set -x
python bench.py --no-cpu-baseline --relabel 0 > gpurun_out/bench_relabel0.log 2>&1
for r in 0 1; do
ncu --kernel-name regex:k_attract_tiled --launch-skip 5 --launch-count 1 --clock-control none \
  --metrics gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,dram__bytes_read.sum,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_active \
  --csv python bench.py --no-cpu-baseline --steps 3 --warmup 3 --relabel $r > gpurun_out/ncu_relabel$r.csv 2>&1
done
