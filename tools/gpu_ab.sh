# parity of the default pipeline + A/B bench against the round-1 backward
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_pinning.py tests/test_gpu_parity.py -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/gpu_tests.log 2>&1
timeout 300 python bench.py --no-extras --no-cpu-baseline --no-e2e --steps 50 > gpurun_out/bench_v2.json 2> gpurun_out/bench_v2.err
TTB_BWD_V2=1 timeout 300 python bench.py --no-extras --no-cpu-baseline --no-e2e --steps 50 > gpurun_out/bench_v1.json 2> gpurun_out/bench_v1.err
tail -5 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log
for f in v1 v2; do python -c "
import json; d=json.loads(open('gpurun_out/bench_$f.json').read()); print('$f', round(d['value']/1e6,1), 'M/s', round(d['ms_per_step']*1e3,1), 'us', {k:v['avg_us'] for k,v in d['kernels'].items()})"; done
