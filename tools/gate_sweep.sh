# gate (auto order) tests + ragged line + cfg2 sweep with the isolated-launch copy reference
timeout 900 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_predict.py -x -q -p no:cacheprovider > gpurun_out/${1}_tests.log 2>&1; echo EXIT $? >> gpurun_out/${1}_tests.log
timeout 300 python bench.py --workload ragged --steps 20 --warmup 3 > gpurun_out/${1}_ragged.json 2>&1
timeout 600 python bench.py --workload sweep --steps 20 --warmup 3 > gpurun_out/${1}_sweep.json 2>&1
