# same-box A/B of two in-tree builds: GNB_LIB=libgnb_base.so (baseline) vs libgnb.so
for rep in 1 2; do
for lib in libgnb_base.so libgnb.so; do
  GNB_LIB=$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-object-api 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib cfg4', d['value'], d['roofline']['frac'])"
  GNB_LIB=$lib timeout 600 python bench.py --workload sweep --steps 20 --warmup 3 2>/dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$lib sweep', [(r['F'], r['frac'], r['frac_of_copy'] if 'frac_of_copy' in r else None) for r in d['rows']])"
done; done
