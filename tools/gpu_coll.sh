set -x
timeout 900 python -m pytest tests/test_gpu_dlrm.py tests/test_gpu_dp.py tests/test_gpu_collection.py -x -q -m gpu > gpurun_out/t.log 2>&1
tail -5 gpurun_out/t.log
timeout 900 python -c "
import json, torch, bench_extras as E
dev = torch.device('cuda', 0)
for name, fn in (('cfg3_native', lambda: E.cfg3(dev)), ('cfg3_permuted', lambda: E.cfg3(dev, permuted=True)), ('cfg4', lambda: E.cfg4(dev)), ('cfg1', lambda: E.cfg1(dev))):
    r = fn(); print(name, json.dumps({k: r[k] for k in r if k in ('value','ms_per_step','per_table_loop')}))
" > gpurun_out/extras.txt 2>&1
cat gpurun_out/extras.txt | tail -8
