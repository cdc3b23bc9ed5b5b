# round-2 profile pass: phase stamps (bwd / plan / fwd), ncu launch list of the config-2 step, full captures
set -x
python -c "import __graft_entry__ as g; g.build()"
python tools/bwd_stamps.py cfg2 > gpurun_out/stamps.txt 2>&1
python tools/bwd_stamps.py cfg3 >> gpurun_out/stamps.txt 2>&1
python tools/plan_stamps.py cfg2 >> gpurun_out/stamps.txt 2>&1
python tools/plan_stamps.py cfg3 >> gpurun_out/stamps.txt 2>&1
python tools/fwd_stamps.py cfg2 >> gpurun_out/stamps.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python tools/prof_fast.py cfg2 3 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fplan|k_fwd|k_bwd|k_coreimg|k_gradcheck" -s 5 -c 5 -o gpurun_out/r2_full_cfg2 -f python tools/prof_fast.py cfg2 3 > gpurun_out/ncu_cfg2.log 2>&1
tail -3 gpurun_out/ncu_cfg2.log
cat gpurun_out/stamps.txt
