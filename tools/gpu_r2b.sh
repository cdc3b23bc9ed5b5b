# round-2 re-entry check: smoke, full GPU suite, full bench line
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/gpu_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -30 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log; tail -c 3000 gpurun_out/bench.json
