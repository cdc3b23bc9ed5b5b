# round-2 first check: smoke, full GPU suite, bench A/B (default backward vs ttb_bwd2)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gpu_tests.log 2>&1
timeout 300 python bench.py --no-extras --no-cpu-baseline --no-e2e --steps 50 > gpurun_out/bench_v1.json 2> gpurun_out/bench_v1.err
TTB_BWD_V2=1 timeout 300 python bench.py --no-extras --no-cpu-baseline --no-e2e --steps 50 > gpurun_out/bench_v2.json 2> gpurun_out/bench_v2.err
TTB_BWD_V2=1 timeout 600 python -m pytest tests/test_gpu_pinning.py -x -q -m gpu > gpurun_out/gpu_tests_v2.log 2>&1
python tools/bwd_stamps.py cfg2 > gpurun_out/stamps.txt 2>&1
TTB_BWD_V2=1 python tools/bwd_stamps.py cfg2 >> gpurun_out/stamps.txt 2>&1
tail -25 gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests_v2.log; tail -2 gpurun_out/smoke.log
for f in v1 v2; do python -c "
import json; d=json.loads(open('gpurun_out/bench_$f.json').read()); print('$f', round(d['value']/1e6,1), 'M/s', round(d['ms_per_step']*1e3,1), 'us', {k:v['avg_us'] for k,v in d['kernels'].items()})"; done
cat gpurun_out/stamps.txt
