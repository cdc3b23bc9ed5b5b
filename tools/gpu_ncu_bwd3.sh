# ncu --set full of the row-grouped backward (config 3), source-level
set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_bwd" -s 1 -c 1 -o gpurun_out/bwd3_full -f python tools/prof_fast.py cfg3 2 > gpurun_out/ncu_bwd3.log 2>&1
tail -2 gpurun_out/ncu_bwd3.log
