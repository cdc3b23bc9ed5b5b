# full default bench (extras, CPU baselines, e2e) + reference arm
set -x
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -3 gpurun_out/bench_full.err; cat gpurun_out/bench_ref.json | cut -c1-300
python -c "
import json; d=json.loads(open('gpurun_out/bench_full.json').read())
print(round(d['value']/1e6,1), 'M/s', 'e2e', round(d['e2e']['value']/1e6,1), 'roof', round(d['roofline']['frac'],3), 'cpu', d['cpu_baseline']['value'])
for k,v in d['extras'].items(): print(k, v.get('value'), v.get('roofline',{}).get('frac'), v.get('cpu_baseline',{}).get('value'), v.get('error'))
"
