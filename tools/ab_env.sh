# same-box A/B of environment knobs on cfg4 + cfg2 sweep: bash tools/ab_env.sh "ENV=.." ...
for rep in 1 2; do
for envs in "$@"; do
  env $envs timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-object-api 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$envs] cfg4', d['value'], d['roofline']['frac'], d['clocks']['reasons'])"
  env $envs timeout 600 python bench.py --workload sweep --steps 20 --warmup 3 2>/dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('[$envs] sweep', [(r['F'], r['frac']) for r in d['rows']])"
done; done
