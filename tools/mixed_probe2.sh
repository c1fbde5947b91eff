# mixed-slot geometry A/B (GNB_MIXED_CFG 0..3) on shuffled / grouped 29-slot and 8-slot batches
N=4194304
timeout 600 python -m pytest tests/test_gpu_mixed.py -x -q -p no:cacheprovider > gpurun_out/probe2_tests.log 2>&1; echo EXIT $? >> gpurun_out/probe2_tests.log
for c in 0 1 2 3; do
  GNB_MIXED_CFG=$c timeout 300 python -m pytest tests/test_gpu_mixed.py -x -q -p no:cacheprovider -k "many_tiles or order_hints" > gpurun_out/probe2_tests_c$c.log 2>&1; echo "cfg $c EXIT $?" >> gpurun_out/probe2_tests_c$c.log
  for S in 29 8; do
    GNB_MIXED_CFG=$c timeout 120 python tools/mixed_probe.py $N 200 $S shuffled | sed "s/^/cfg$c /"
    GNB_MIXED_CFG=$c GNB_PRED_MIXED=2 timeout 120 python tools/mixed_probe.py $N 200 $S grouped | sed "s/^/cfg$c forced /"
  done
done
