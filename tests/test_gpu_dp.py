"""Data-parallel step on the CUDA path, world size 2 on one GPU (gloo moves
the CUDA gradient buffer; NCCL needs one GPU per rank): every rank plans,
forwards and backwards its bag shard with the tensor-core pipeline, the flat
core gradients are all-reduced, every rank applies ttb_sgd_update. After
three steps both replicas are bitwise identical and equal the single-process
run on the whole batch (tolerance: fp32 reduction order)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

GEOM = ((20, 20, 25), (4, 4, 4), (1, 32, 32, 1))
STEPS, LR, MU = 3, 0.05, 0.9


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batches():
    rng = np.random.default_rng(17)
    out = []
    for _ in range(STEPS):
        sizes = rng.integers(1, 4, size=600)
        idx = rng.integers(0, 10_000, size=int(sizes.sum()))
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        gout = (rng.standard_normal((600, 64)) / 600).astype(np.float32)
        out.append((idx, off, gout))
    return out


def _run(rank, world):
    from oracle import ttb_oracle as O
    from paper_2507_14668_b200 import dp
    from paper_2507_14668_b200.engine import TtEngine
    from paper_2507_14668_b200.geometry import TtShape
    shape = TtShape(*GEOM)
    g = O.Geometry(*GEOM)
    cores = [torch.from_numpy(c.astype(np.float32)).cuda() for c in O.init_cores(g, 2)]
    flat = dp.FlatCores(cores, device="cuda")
    eng = TtEngine(shape, 4096, 1024, "cuda")
    assert eng.fast
    for idx, off, gout in _batches():
        ti, to = torch.from_numpy(idx).cuda(), torch.from_numpy(off).cuda()
        li, lo, (b0, b1) = dp.local_batch(ti, to, rank, world)
        dp.dp_step(eng, flat, li, lo, torch.from_numpy(gout[b0:b1]).cuda(), LR, MU)
    torch.cuda.synchronize()
    return flat.param.cpu().numpy()


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _run(rank, world)))
    finally:
        dist.destroy_process_group()


def test_dp_ws2_matches_single_process():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(res[0][1], res[1][1])  # replicas identical after every update
    want = _run(0, 1)  # one process, whole batch
    err = np.abs(res[0][1] - want).max() / np.abs(want).max()
    assert err < 1e-5, err


def _dlrm_run(rank, world):
    from paper_2507_14668_b200.model import DlrmModel, ModelConfig
    torch.backends.cuda.matmul.allow_tf32 = False
    cfg = ModelConfig(n_dense=5, rows_per_field=(10_000, 300, 2_000), emb_dim=64, ranks=(1, 32, 32, 1),
                      tt_threshold=1000, bottom_sizes=(32,), top_sizes=(32,), loss="bce", seed=3)
    model = DlrmModel(cfg, max_indices=4096)
    rng = np.random.default_rng(9)
    B = 512
    for _ in range(STEPS):
        dense = rng.standard_normal((B, 5)).astype(np.float32)
        labels = (rng.random(B) < 0.3).astype(np.float64)
        sparse = []
        for rows in cfg.rows_per_field:
            sizes = rng.integers(1, 3, size=B)
            idx = rng.integers(0, rows, size=int(sizes.sum()))
            off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
            b0, b1 = (B * rank) // world, (B * (rank + 1)) // world
            sparse.append((torch.from_numpy(idx[off[b0]:off[b1]]).cuda(),
                           torch.from_numpy(off[b0:b1 + 1] - off[b0]).cuda()))
        b0, b1 = (B * rank) // world, (B * (rank + 1)) // world
        model.train_step_dp(torch.from_numpy(dense[b0:b1]).cuda(), sparse, torch.from_numpy(labels[b0:b1]).cuda(),
                            0.05, 0.9, global_batch=B)
    torch.cuda.synchronize()
    return np.concatenate([p.detach().cpu().numpy().reshape(-1) for _, p in model.named_ref_params()])


def _dlrm_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _dlrm_run(rank, world)))
    finally:
        dist.destroy_process_group()


def test_dlrm_dp_ws2_matches_single_process():
    """BASELINE config 5's step (data-parallel TT-DLRM: one flat all-reduce of
    TT-core, dense-field and MLP gradients, batch-mean scaling, identical
    update on every rank), world size 2 on one GPU, against one process on
    the whole batch."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dlrm_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(res[0][1], res[1][1])
    want = _dlrm_run(0, 1)
    err = np.abs(res[0][1] - want).max() / np.abs(want).max()
    assert err < 1e-5, err
