# A/B of row-box K-PRED knobs (GNB_ROWBOX_BULK, GNB_ROWBOX_CVT) on cfg2-style shapes.
set -u
python -m pytest tests/test_gpu_predict.py -x -q > gpurun_out/gputests.log 2>&1; echo tests $?
for bulk in 1 0; do
  for r in 16000000 1000000; do
    for F in 50 100; do
    GNB_ROWBOX_BULK=$bulk python bench.py --rows $r --features $F --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bulk=$bulk rows=$r F=$F', d['value'], d['roofline']['frac'])"
    done
  done
  GNB_ROWBOX_BULK=$bulk python bench.py --workload sweep --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bulk=$bulk sweep', [(r['F'], r['frac']) for r in d['rows']])"
done
