# quick iteration: parity subset, stamps, bench (no extras)
set -x
timeout 600 python -m pytest tests/test_gpu_pinning.py tests/test_gpu_parity.py -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/gpu_tests.log 2>&1
python tools/bwd_stamps.py cfg2 > gpurun_out/stamps.txt 2>&1
python tools/bwd_stamps.py cfg3 >> gpurun_out/stamps.txt 2>&1
timeout 300 python bench.py --no-extras --no-cpu-baseline --no-e2e --steps 50 > gpurun_out/bench_v2.json 2> gpurun_out/bench_v2.err
tail -3 gpurun_out/gpu_tests.log; cat gpurun_out/stamps.txt
python -c "
import json; d=json.loads(open('gpurun_out/bench_v2.json').read()); print('v2', round(d['value']/1e6,1), 'M/s', round(d['ms_per_step']*1e3,1), 'us', {k:v['avg_us'] for k,v in d['kernels'].items()})"
