# ncu launch list + full captures of the step kernels (config 2), bench without extras
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_fast.py cfg2 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bwd|k_fwd|k_coreimg|k_sgd3" -s 8 -c 4 -o gpurun_out/full_cfg2 -f python tools/prof_fast.py cfg2 4 > gpurun_out/ncu_full.log 2>&1
python -m pytest tests -m gpu -q -rs 2>&1 | grep -i skip > gpurun_out/skips.txt
