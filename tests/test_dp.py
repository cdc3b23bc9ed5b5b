"""Data-parallel host logic on CPU with gloo, world size 2: bag sharding,
flat buffers and the gradient all-reduce give the single-process gradient of
the whole batch (core gradients are additive), and every rank ends with the
same update. Per-shard gradients come from the oracle (test checker only)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ttb_oracle as O
from paper_2507_14668_b200 import dp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    g = O.Geometry((6, 7, 9), (2, 2, 4), (1, 4, 5, 1))
    cores = [c.astype(np.float32) for c in O.init_cores(g, 3)]
    rng = np.random.default_rng(5)
    sizes = rng.integers(1, 5, size=37)
    idx = rng.integers(0, g.rows, size=int(sizes.sum()))
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    gout = rng.standard_normal((37, g.cols)).astype(np.float32)
    return g, cores, idx, off, gout


def _grads(g, cores, idx, off, gout):
    rows, ug = O.unique_aggregate(idx, np.repeat(gout.astype(np.float64), np.diff(off), axis=0))
    return O.core_grads([c.astype(np.float64) for c in cores], g, rows, ug)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g, cores, idx, off, gout = _problem()
        ti, to = torch.from_numpy(idx), torch.from_numpy(off)
        li, lo, (b0, b1) = dp.local_batch(ti, to, rank, world)
        flat = dp.FlatCores([torch.from_numpy(c) for c in cores], device="cpu")
        local = _grads(g, cores, li.numpy(), lo.numpy(), gout[b0:b1])
        for v, gk in zip(flat.grads, local):
            v.copy_(torch.from_numpy(gk.astype(np.float32)))
        dp.allreduce_grads(flat.grad)
        # the update every rank applies (same numbers on every rank)
        p = flat.param.double() - 0.05 * flat.grad.double()
        q.put((rank, flat.grad.numpy().copy(), p.float().numpy()))
    finally:
        dist.destroy_process_group()


def test_shard_bags_cover_batch():
    off = torch.tensor([0, 2, 3, 7, 8, 11, 12])
    seen = []
    for r in range(4):
        b0, b1, t0, t1 = dp.shard_bags(off, r, 4)
        seen.extend(range(b0, b1))
        assert t0 == int(off[b0]) and t1 == int(off[b1])
    assert seen == list(range(6))
    li, lo, _ = dp.local_batch(torch.arange(12), off, 1, 2)
    assert lo[0] == 0 and lo[-1] == li.numel()


def test_flat_views_alias_buffers():
    cores = [torch.ones(1, 6, 2), torch.full((2, 8, 3), 2.0), torch.full((3, 4, 1), 3.0)]
    fc = dp.FlatCores(cores, device="cpu")
    assert fc.param.numel() == 12 + 48 + 12
    fc.grads[1].fill_(7.0)
    assert float(fc.grad[12:60].sum()) == 7.0 * 48
    assert fc.velocity.dtype == torch.float64


@pytest.mark.timeout(120)
def test_allreduce_equals_full_batch_gradient_gloo_ws2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=90) for _ in range(world))
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    g, cores, idx, off, gout = _problem()
    full = _grads(g, cores, idx, off, gout)
    want = np.concatenate([x.reshape(-1) for x in full])
    for rank, grad, _ in res:
        err = np.abs(grad - want).max() / np.abs(want).max()
        assert err < 1e-5, (rank, err)
    assert np.array_equal(res[0][1], res[1][1])  # identical reduced gradient on every rank
    assert np.array_equal(res[0][2], res[1][2])  # hence identical replicas after the step
