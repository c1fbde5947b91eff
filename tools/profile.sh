#!/bin/bash
# Profiling recipe (B200_PROFILING.md): plain run first, then the ncu launch list,
# then one --set full capture of each of our kernels.  Run under gpurun.
set -u
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:predict_tma -s 3 -c 1 \
    -o gpurun_out/prof_predict -f $CMD > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fit_tma -c 1 \
    -o gpurun_out/prof_fit -f $CMD > gpurun_out/ncu_fit.log 2>&1
echo done
