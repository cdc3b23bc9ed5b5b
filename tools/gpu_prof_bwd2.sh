# per-phase stamps + one ncu --set full capture of the v2 backward (config 2)
set -x
python tools/bwd_stamps.py cfg2 > gpurun_out/stamps.txt 2>&1
python tools/bwd_stamps.py cfg3 >> gpurun_out/stamps.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_bwd2 -c 1 -o gpurun_out/bwd2_cfg2 python tools/prof_fast.py cfg2 2 > gpurun_out/ncu_bwd2.log 2>&1
cat gpurun_out/stamps.txt
