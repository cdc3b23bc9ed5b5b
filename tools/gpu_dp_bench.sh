# bench.py's N > 1 path on one GPU: two ranks over gloo (NCCL needs one GPU per rank)
set -x
python -c "import __graft_entry__ as g; g.build()"
TTB_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_dp2.json 2> gpurun_out/bench_dp2.err
timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 20 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
tail -3 gpurun_out/bench_dp2.err
