# round-end evidence: full bench (+extras, cpu baseline), reference arm, ncu launch list and full captures
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fast.csv python tools/prof_fast.py cfg2 3 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fplan|k_fwd|k_bwd|k_coreimg" -s 4 -c 4 -o gpurun_out/full_fast -f python tools/prof_fast.py cfg2 3 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/gpu_tests.log
