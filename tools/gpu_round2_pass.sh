set -x
python -m pytest tests -m gpu -x -q -p no:cacheprovider -rs > gpurun_out/r02_gpu_tests_2.log 2>&1; echo EXIT $? >> gpurun_out/r02_gpu_tests_2.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_n1.json 2> gpurun_out/r02_bench_n1.err
python bench.py --workload sweep --steps 20 --warmup 3 > gpurun_out/r02_bench_sweep.json 2>&1
python bench.py --workload ragged --steps 20 --warmup 3 > gpurun_out/r02_bench_ragged.json 2>&1
python bench.py --workload fit --steps 5 --warmup 3 > gpurun_out/r02_bench_fit.json 2>&1
python bench.py --workload fin --steps 5 --warmup 3 > gpurun_out/r02_bench_fin.json 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_ref.json 2>&1
tail -3 gpurun_out/r02_gpu_tests_2.log
