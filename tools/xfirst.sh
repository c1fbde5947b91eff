timeout 900 python -m pytest tests/test_gpu_predict.py tests/test_gpu_fuzz.py tests/test_gpu_mixed.py tests/test_gpu_api.py -x -q -p no:cacheprovider > gpurun_out/${1}_tests.log 2>&1; echo EXIT $? >> gpurun_out/${1}_tests.log
timeout 600 python bench.py --workload sweep --steps 20 --warmup 3 > gpurun_out/${1}_sweep.json 2>&1
timeout 300 python bench.py --workload ragged --steps 20 --warmup 3 > gpurun_out/${1}_ragged.json 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-object-api > gpurun_out/${1}_cfg4.json 2>&1
