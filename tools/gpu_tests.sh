# build, the GPU suite (durations), smoke and a quick bench
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=15 ${PYTEST_ARGS} > gpurun_out/gpu_tests.log 2>&1
timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 50 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
tail -25 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log
