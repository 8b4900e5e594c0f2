#!/bin/bash
# Round-2 final profiling pass (run under gpurun, one GPU):
#   launch list of a short default bench (C3 + sub-records) and one
#   ncu --set full capture each of kernel (a)+(b) (C3) and of E1 (C4 20k).
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-sim --no-emit --no-api --no-cfg"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02f.csv $CMD > /dev/null 2>&1 || true
ncu --set full --import-source on --clock-control none -k regex:'mfp_phase|requirements_kernel|compact_list' \
    -c 3 -o gpurun_out/c3_full_r02f python scripts/one_solve_req.py > gpurun_out/ncu_c3_r02f.log 2>&1 || true
ncu --set full --import-source on --clock-control none -k regex:'replay_kernel|region_kernel' \
    -c 2 -o gpurun_out/c4_full_r02f python scripts/one_replay.py 20000 > gpurun_out/ncu_c4_r02f.log 2>&1 || true
ls -la gpurun_out
