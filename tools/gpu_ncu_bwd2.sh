set -x
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_bwd2 -c 1 -o gpurun_out/bwd2_cfg2 -f python tools/prof_fast.py cfg2 2 > gpurun_out/ncu_bwd2.log 2>&1
tail -3 gpurun_out/ncu_bwd2.log
