# build, GPU tests, bench (no extras) and a launch list
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_fast.py cfg2 3 > /dev/null 2>&1
tail -3 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log
