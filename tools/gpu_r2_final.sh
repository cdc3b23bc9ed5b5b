# round-2 evidence: smoke, full GPU suite, full bench, reference arm, ncu launch list + full captures (cfg2, cfg3)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_launches_cfg2.csv python tools/prof_fast.py cfg2 3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_launches_cfg3.csv python tools/prof_fast.py cfg3 2 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fplan|k_fwd|k_bwd|k_coreimg" -s 4 -c 4 -o gpurun_out/r2_full_cfg2 -f python tools/prof_fast.py cfg2 3 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fwd|k_bwd|k_rowsort" -s 3 -c 3 -o gpurun_out/r2_full_cfg3 -f python tools/prof_fast.py cfg3 2 > gpurun_out/ncu_full3.log 2>&1
tail -3 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log
