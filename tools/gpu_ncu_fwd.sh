# ncu --set full of the forward kernel only (config 2), source-level
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_fwd" -s 1 -c 1 -o gpurun_out/fwd_full -f python tools/prof_fast.py cfg2 3 > gpurun_out/ncu_fwd.log 2>&1
tail -3 gpurun_out/ncu_fwd.log
