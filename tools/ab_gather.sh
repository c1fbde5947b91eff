# A/B of K-PRED geometry / L2 promotion on the cfg3 ragged workload
# (grouped rows and slot-sorted shuffled rows): bash tools/ab_gather.sh "ENV=.." ...
for envs in "$@"; do
  env $envs python bench.py --workload ragged --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$envs', 'grouped', d['frac'], 'sorted', d['shuffled_rows_slot_sorted']['value'], d['shuffled_rows_slot_sorted']['frac'], d['shuffled_rows_slot_sorted']['labels_equal_unsorted_path'])"
done
