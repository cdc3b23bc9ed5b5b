# config-3 iteration: parity subset, per-kernel times (one table, and the 26-table batched handle)
set -x
timeout 300 python -m pytest tests/test_gpu_pinning.py tests/test_gpu_parity.py tests/test_gpu_collection.py -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/it3_tests.log 2>&1
for w in cfg2 cfg3 cfg3p; do timeout 120 python tools/cfg_kernels.py $w; done > gpurun_out/it3_kernels.txt 2>&1
for w in native permuted; do timeout 120 python tools/cfg3_batched_kernels.py $w; done >> gpurun_out/it3_kernels.txt 2>&1
tail -5 gpurun_out/it3_tests.log; cat gpurun_out/it3_kernels.txt
