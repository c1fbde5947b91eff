# A/B of L2 promotion / gather boxes on the cfg3 ragged workload (grouped and slot-sorted shuffled rows)
for envs in "GNB_L2_PROMO=3" "GNB_L2_PROMO=0" "GNB_L2_PROMO=1" "GNB_L2_PROMO=2" "GNB_L2_PROMO=0 GNB_GATHER_B=2"; do
  env $envs python bench.py --workload ragged --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$envs', 'grouped', d['frac'], 'sorted', d['shuffled_rows_slot_sorted']['value'], d['shuffled_rows_slot_sorted']['frac'], d['shuffled_rows_slot_sorted']['labels_equal_unsorted_path'])"
done
