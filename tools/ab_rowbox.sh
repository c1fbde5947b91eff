# A/B of row-box K-PRED knobs on cfg2-style shapes: bash tools/ab_rowbox.sh "ENV=.. ENV2=.." ...
set -u
python -m pytest tests/test_gpu_predict.py tests/test_gpu_api.py -x -q > gpurun_out/gputests.log 2>&1; echo tests $?
for envs in "$@"; do
  for r in 16000000 1000000; do
    for F in 50 100; do
    env $envs python bench.py --rows $r --features $F --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$envs rows=$r F=$F', d['value'], d['roofline']['frac'])"
    done
  done
  env $envs python bench.py --workload sweep --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$envs sweep', [(r['F'], r['frac']) for r in d['rows']])"
done
