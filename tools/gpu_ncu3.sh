# config-3 source-level ncu of the step kernels (one table) + stamps + ablations
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_fwd|k_bwd" -s 2 -c 2 -o gpurun_out/it3 -f python tools/prof_fast.py cfg3 2 > gpurun_out/ncu_it3.log 2>&1
bash tools/bwd_ablate3.sh > gpurun_out/ablate3.txt 2>&1
tail -3 gpurun_out/ncu_it3.log; cat gpurun_out/ablate3.txt | grep -v Warn
