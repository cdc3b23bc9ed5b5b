# A/B of the config-2 bench step: ab/libttb_base.so against the tree's libttb.so, alternating, same box
for r in 1 2 3; do
  for v in base new; do
    if [ $v = base ]; then export TTB_LIB_PATH=ab/libttb_base.so; else unset TTB_LIB_PATH; fi
    python bench.py --no-extras --no-cpu-baseline --no-e2e --steps 200 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,1), {k:v['avg_us'] for k,v in d['kernels'].items()})"
  done
done
