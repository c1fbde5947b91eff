# Full GPU pass: tests, smoke, default bench, reference arm, every workload line,
# ncu launch list of the bench (cold, serialised -- only the kernel's SHARE of
# the step counts) and one ncu --set full capture of the mixed-slot kernel.
set -x
tag=${1:-r02}
python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/${tag}_gpu_tests.log 2>&1; echo EXIT $? >> gpurun_out/${tag}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo EXIT $? >> gpurun_out/${tag}_smoke.log
python bench.py > gpurun_out/${tag}_bench_n1.json 2> gpurun_out/${tag}_bench_n1.err
python bench.py --impl reference > gpurun_out/${tag}_bench_ref.json 2>&1
for w in sweep ragged fit fin; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 3 > gpurun_out/${tag}_bench_$w.json 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 3 --warmup 3 \
    --no-cpu-baseline --no-object-api > gpurun_out/${tag}_ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:predict_mixed -s 3 -c 1 \
    -o gpurun_out/${tag}_mixed_shuf29 python tools/mixed_probe.py 4194304 200 29 shuffled > gpurun_out/${tag}_ncu_mixed.log 2>&1
tail -3 gpurun_out/${tag}_gpu_tests.log
