#!/bin/bash
# GPU-box profiling pass for configuration C3 (run under gpurun):
#   1. the bench line (no profiler)
#   2. the ncu launch list of a short bench run (per-kernel shares)
#   3. one ncu --set full capture of both kernel-(a) phase launches and kernel (b)
set -e
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
CMD="python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $CMD > /dev/null 2>&1 || true
ncu --set full --import-source on --clock-control none -k regex:'mfp_phase|requirements_kernel|compact_list' \
    -c 3 -o gpurun_out/c3_full python scripts/one_solve_req.py > gpurun_out/ncu_full.log 2>&1 || true
