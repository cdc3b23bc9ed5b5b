# ncu --set full of the step kernels (config 2 and config 3), source-level
set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fplan|k_fwd|k_bwd|k_coreimg|k_gradcheck" -s 5 -c 5 -o gpurun_out/r2_full_cfg2 -f python tools/prof_fast.py cfg2 3 > gpurun_out/ncu_cfg2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fwd|k_bwd" -s 2 -c 2 -o gpurun_out/r2_full_cfg3 -f python tools/prof_fast.py cfg3 2 > gpurun_out/ncu_cfg3.log 2>&1
tail -3 gpurun_out/ncu_cfg2.log gpurun_out/ncu_cfg3.log
