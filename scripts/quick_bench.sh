# quick C2 step + per-op breakdown (10 steps, no CPU baseline)
python bench.py --no-cpu --steps 10 "$@" 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read())
print(d['ms_per_step'], d['speedup_vs_nodedup'], d['clocks']['sm_mhz'], {k:v['us_per_step'] for k,v in d['breakdown_us_radix'].items()})"
