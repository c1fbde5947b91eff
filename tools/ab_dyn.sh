timeout 900 python -m pytest tests/test_gpu_predict.py tests/test_gpu_fuzz.py tests/test_gpu_mixed.py tests/test_gpu_api.py tests/test_gpu_sharded.py -x -q -p no:cacheprovider 2>&1 | tail -2 > gpurun_out/dyn_tests.log
LIBS="libgnb_base.so libgnb.so" bash tools/ab_lib3.sh > gpurun_out/dyn_ab.log 2>&1
for lib in libgnb_base.so libgnb.so; do GNB_LIB=$lib timeout 300 python bench.py --workload ragged --steps 20 --warmup 3 2>/dev/null | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib ragged', d['frac'], d['shuffled_rows']['frac'], d['shuffled_rows_slot_sorted']['frac'])"; done >> gpurun_out/dyn_ab.log
