"""The fused data-parallel exchange kernel (ttb_dp_exchange_update,
csrc/ttb_dp.cu): reduce-scatter -> update of the owned shard -> all-gather
over peer memory, one kernel per rank. On one GPU the W ranks are W buffer
sets in one process, their kernels launched concurrently on W streams (they
synchronise through the flag words exactly as ranks on W GPUs do); the CUDA
IPC mapping used across processes is checked with two processes (gloo).
Expected values: the reference's update rule on the summed gradient
(fused_update, backward.py:186-204 via the oracle's sgd_step / adagrad_step)
with the sum taken in fp64 in peer order and rounded once."""
import ctypes
import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import ttb_oracle as O

pytestmark = pytest.mark.gpu


def run_ranks(params, grads, states, lr, mu, adagrad=False, errs=None, steps=1):
    from paper_2507_14668_b200 import _native as nat
    from paper_2507_14668_b200.dp import make_peers
    from paper_2507_14668_b200.engine import _ptr
    lib = nat.load()
    W = len(params)
    flags = [torch.zeros(int(lib.ttb_dp_flag_words(W)), dtype=torch.int32, device="cuda") for _ in range(W)]
    table = [(_ptr(grads[r]), _ptr(params[r]), _ptr(flags[r])) for r in range(W)]
    streams = [torch.cuda.Stream() for _ in range(W)]
    torch.cuda.synchronize()
    for _ in range(steps):
        for r in range(W):
            P = make_peers(r, table)
            with torch.cuda.stream(streams[r]):
                nat.check(lib.ttb_dp_exchange_update(
                    ctypes.byref(P), params[r].numel(),
                    lr, mu, int(adagrad), _ptr(states[r]) if states[r] is not None else None,
                    _ptr(errs[r]) if errs is not None else None, 8, torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
    return flags


@pytest.mark.parametrize("W", [2, 3])
@pytest.mark.parametrize("adagrad", [False, True])
def test_exchange_matches_update_of_summed_grads(W, adagrad):
    rng = np.random.default_rng(W + 10 * adagrad)
    n = 100_003
    p0 = rng.standard_normal(n).astype(np.float32)
    gs = [rng.standard_normal(n).astype(np.float32) for _ in range(W)]
    params = [torch.from_numpy(p0.copy()).cuda() for _ in range(W)]
    grads = [torch.from_numpy(g).cuda() for g in gs]
    states = [torch.zeros(n, dtype=torch.float64, device="cuda") for _ in range(W)]
    flags = run_ranks(params, grads, states, 0.05, 1e-10 if adagrad else 0.9, adagrad, steps=2)
    total = np.zeros(n)
    for g in gs:
        total += g.astype(np.float64)
    g32 = total.astype(np.float32)
    want, st = p0.copy(), None
    for _ in range(2):
        st = O.adagrad_step(want, g32, 0.05, 1e-10, st) if adagrad else O.sgd_step(want, g32, 0.05, 0.9, st)
    for r in range(W):
        assert np.array_equal(params[r].cpu().numpy(), want), r  # every replica, bit for bit
    owned = np.concatenate([states[r].cpu().numpy()[n * r // W: n * (r + 1) // W] for r in range(W)])
    assert np.array_equal(owned, st)
    assert all(int(f[2 * W + 1]) == 2 for f in flags)  # epoch advanced once per call


def test_exchange_bad_rank_cancels_everywhere():
    W, n = 2, 5000
    params = [torch.ones(n, device="cuda") for _ in range(W)]
    grads = [torch.ones(n, device="cuda") for _ in range(W)]
    errs = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(W)]
    errs[1][0] = 8  # rank 1's local finiteness check failed
    run_ranks(params, grads, [None] * W, 0.1, 0.0, errs=errs)
    for r in range(W):
        assert torch.equal(params[r], torch.ones(n, device="cuda"))
        assert int(errs[r][0]) & 8


def _ipc_worker(rank, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    from paper_2507_14668_b200.dp import PeerExchange
    from paper_2507_14668_b200 import _native as nat
    from paper_2507_14668_b200.engine import _ptr, _stream
    lib = nat.load()
    torch.cuda.set_device(0)
    pad = torch.zeros(37, device="cuda")  # the buffers do not start an allocation
    param = torch.full((1000,), float(rank + 1), device="cuda")
    grad = torch.full((1000,), 10.0 * (rank + 1), device="cuda")
    ex = PeerExchange(param, grad)
    dist.barrier()
    if rank == 1:  # through the mapping: rank 0's params -= 1.0 * rank 1's grads
        peer = ex.peers.param[0]
        nat.check(lib.ttb_sgd_update(peer, _ptr(grad), None, 1000, 1.0, 0.0, _stream()))
        torch.cuda.synchronize()
    dist.barrier()
    if rank == 0:
        q.put(param.cpu().numpy().tolist())
    dist.barrier()
    ex.close()
    del pad
    dist.destroy_process_group()


def test_ipc_mapping_two_processes():
    """PeerExchange maps the other process's buffers: rank 1 updates rank 0's
    parameters in place through the mapped pointer (the same device here)."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_ipc_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = q.get(timeout=300)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got == [1.0 - 20.0] * 1000
