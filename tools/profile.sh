#!/bin/bash
# Profiling recipe (B200_PROFILING.md): plain run first, then the ncu launch list,
# then one --set full capture of each of our hot kernels.  Run under gpurun:
#   gpurun -- 'bash tools/profile.sh'
set -u
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
mkdir -p gpurun_out
timeout 600 $CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
# int32 K-PRED (4th launch: after 3 warm-ups), then the uint8 launch of the same run
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:predict_tma_kernel -s 3 -c 1 -o gpurun_out/prof_predict -f $CMD \
    > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"predict_tma_kernel<2, unsigned char" -c 1 -o gpurun_out/prof_predict_u8 -f $CMD \
    > gpurun_out/ncu_u8.log 2>&1
FIT="python bench.py --workload fit --fit-rows 100000000"
timeout 600 $FIT > gpurun_out/plain_fit.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fit_tma -s 1 -c 1 \
    -o gpurun_out/prof_fit16 -f $FIT > gpurun_out/ncu_fit16.log 2>&1
echo done
