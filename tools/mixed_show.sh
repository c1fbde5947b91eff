tag=$1
tail -3 gpurun_out/${tag}_tests.log; cat gpurun_out/${tag}_debug.log | grep mismatch
for m in 1 0; do python -c "
import json
for l in open('gpurun_out/${tag}_ragged_m$m.json'):
    if l.startswith('{'):
        d=json.loads(l); print('m$m grouped', d['frac'], d['ms'], d['bit_exact_subsample_vs_oracle'], 'shuffled', d['shuffled_rows']['frac'], d['shuffled_rows']['bit_exact_vs_grouped_order'], 'sorted', d['shuffled_rows_slot_sorted']['frac'])
"; done; grep -o '"value": [0-9.]*' gpurun_out/${tag}_cfg4_m2.json | head -1
