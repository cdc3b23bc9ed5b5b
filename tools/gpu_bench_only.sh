# full bench line (with extras, CPU baselines) and the reference arm
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
