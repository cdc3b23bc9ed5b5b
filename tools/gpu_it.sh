# quick iteration: parity subset, backward stamps, bench (no extras)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_pinning.py tests/test_gpu_parity.py -x -q ${PYTEST_ARGS} > gpurun_out/it_tests.log 2>&1
python tools/bwd_stamps.py cfg2 > gpurun_out/it_stamps.txt 2>&1
timeout 300 python bench.py --no-extras --no-cpu-baseline --no-e2e --steps 100 > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err
tail -5 gpurun_out/it_tests.log; cat gpurun_out/it_stamps.txt
python -c "
import json; d=json.loads(open('gpurun_out/it_bench.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,1), 'M/s', round(d['ms_per_step']*1e3,1), 'us', {k:v['avg_us'] for k,v in d['kernels'].items()}, d['roofline']['frac'])"
