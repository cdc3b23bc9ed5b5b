# quick A/B on one box: parity subset with the tree's library, then the config-2 bench step and
# per-kernel times (cfg2 / cfg3) for ab/libttb_base.so against the tree's libttb.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pinning.py tests/test_gpu_adagrad.py tests/test_gpu_collection.py -m gpu -q -x > gpurun_out/ab_tests.log 2>&1
tail -2 gpurun_out/ab_tests.log
bash tools/ab_bench.sh 2>&1 | tee gpurun_out/ab_bench.log
for v in base new base new; do
  if [ $v = base ]; then export TTB_LIB_PATH=ab/libttb_base.so; else unset TTB_LIB_PATH; fi
  for c in cfg2 cfg3; do echo "$v $(timeout 300 python tools/cfg_kernels.py $c 2>&1 | tail -1)"; done
done 2>&1 | tee gpurun_out/ab_kernels.log
timeout 200 python tools/fwd_stamps.py 2>&1 | tail -6 > gpurun_out/fwd_stamps_new.txt
