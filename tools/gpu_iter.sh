# quick iteration: parity subset, stamps, bench (no extras), optional ncu of one kernel ($NCU_K)
set -x
timeout 900 python -m pytest tests/test_gpu_pinning.py tests/test_gpu_parity.py tests/test_gpu_ops.py -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/gpu_tests.log 2>&1
python tools/bwd_stamps.py cfg2 > gpurun_out/stamps.txt 2>&1
timeout 300 python bench.py --no-extras --no-cpu-baseline --no-e2e --steps 50 > gpurun_out/bench_it.json 2> gpurun_out/bench_it.err
if [ -n "$NCU_K" ]; then timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$NCU_K" -s 2 -c 1 -o gpurun_out/it -f python tools/prof_fast.py ${NCU_CFG:-cfg2} 3 > gpurun_out/ncu_it.log 2>&1; fi
tail -5 gpurun_out/gpu_tests.log; cat gpurun_out/stamps.txt; tail -3 gpurun_out/bench_it.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_it.json').read()); print(round(d['value']/1e6,1), 'M/s', round(d['ms_per_step']*1e3,1), 'us', {k:v['avg_us'] for k,v in d['kernels'].items()})"
