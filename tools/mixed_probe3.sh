# mixed-slot kernel: tests + shuffled probes + ragged bench line
N=4194304
[ -n "$TESTS" ] && timeout 900 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_predict.py -x -q -p no:cacheprovider > gpurun_out/${1}_tests.log 2>&1; echo EXIT $? >> gpurun_out/${1}_tests.log
[ -n "$TESTS" ] && timeout 300 python tools/mixed_debug.py 4194304 > gpurun_out/${1}_debug.log 2>&1
for S in 29 8 2; do timeout 120 python tools/mixed_probe.py $N 200 $S shuffled; done
timeout 300 python bench.py --workload ragged --steps 20 --warmup 3 > gpurun_out/${1}_ragged.json 2>&1
if [ -n "$NCU" ]; then
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:predict_mixed -s 3 -c 1 \
    -o gpurun_out/${1}_shuf29 python tools/mixed_probe.py $N 200 29 shuffled > gpurun_out/${1}_ncu.log 2>&1
fi
