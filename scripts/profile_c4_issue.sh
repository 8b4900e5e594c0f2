#!/bin/bash
# Issue-rate evidence for E1 (replay_kernel) on the C4 batch: one ncu capture
# of the first replay launch of `bench.py --workload c4` (100k functions),
# summarised into profiles/c4_issue.json by scripts/summarize_c4_issue.py.
set -e
mkdir -p gpurun_out
ncu --kernel-name regex:replay_kernel --launch-count 1 --clock-control none \
  --metrics sm__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second \
  --csv --log-file gpurun_out/c4_issue.csv \
  python bench.py --workload c4 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-parity > gpurun_out/c4_issue_bench.log 2>&1
