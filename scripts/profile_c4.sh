#!/bin/bash
# GPU-box profiling pass for configuration C4 (run under gpurun): the ncu
# launch list of a short device-resident E1 run over 20k functions, and one
# ncu --set full capture of the E1 replay kernel (region table + replay).
mkdir -p gpurun_out
CMD="python bench.py --workload c4 --c4-funcs 20000 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $CMD > /dev/null 2>&1 || true
ncu --set full --import-source on --clock-control none -k regex:'replay_kernel|region_kernel' \
    -c 2 -o gpurun_out/c4_full $CMD > gpurun_out/ncu_c4_full.log 2>&1 || true
