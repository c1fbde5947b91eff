# Mixed-slot K-PRED A/B on cfg3 (ragged, F=200, 29 slots): grouped + shuffled
# rows with the mixed kernel (default), without it (GNB_PRED_MIXED=0: 6-CTA
# kernel, slot sort + gather4 for the shuffled batch), and forced for one slot.
set -x
tag=${1:-mixed}
timeout 900 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_predict.py tests/test_gpu_api.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1; echo EXIT $? >> gpurun_out/${tag}_tests.log
timeout 300 python tools/mixed_debug.py 4194304 > gpurun_out/${tag}_debug.log 2>&1
for m in 1 0; do
  GNB_PRED_MIXED=$m timeout 300 python bench.py --workload ragged --steps 20 --warmup 3 > gpurun_out/${tag}_ragged_m$m.json 2>&1
done
GNB_PRED_MIXED=2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-object-api > gpurun_out/${tag}_cfg4_m2.json 2>&1
if [ -n "$NCU" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:predict_mixed -s 26 -c 1 \
    -o gpurun_out/${tag}_mixed python bench.py --workload ragged --steps 20 --warmup 3 > gpurun_out/${tag}_ncu.log 2>&1
fi
tail -2 gpurun_out/${tag}_tests.log
