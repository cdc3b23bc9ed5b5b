# ncu launch list (serialised, cold) of a few config-2 steps: gpurun_out/launches.csv
python -c "import __graft_entry__ as g; g.build()"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_fast.py ${WL:-cfg2} 3 > /dev/null 2>&1
