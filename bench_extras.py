"""Secondary BASELINE configs measured by bench.py (reported under "extras").

    cfg1  Reference CPU Rec-AD DLRM: one TT field 1M x 16, ranks 16, batch 256,
          FDIA-style bags of 1-3 Zipf(1.05) indices             -> samples/s
    cfg3  26 TT tables 10M x 64, ranks 32, Zipf(1.05), pooling 20,
          B = 65,536 bags per table, native and permuted ids     -> lookups/s
    cfg4  Criteo-Kaggle-shaped TT-DLRM (13 dense, 26 sparse, 15 TT fields at
          tt_threshold 1000), bottom 512-256-64, top 512-256-1,
          B = 65,536, fp32 MLPs (TF32 off)                       -> samples/s

Every step runs through the public API (TTEmbeddingBag / DlrmModel) and is
replayed as one CUDA graph; timings are CUDA events over the timed steps.
Synthetic data: Zipf by inverse CDF (same law as the reference's
rng.choice(p=zipf_probs), data.py:103-108, 164; different random stream).
"""
from __future__ import annotations

import numpy as np
import torch

KAGGLE_ROWS = (1460, 583, 10131227, 2202608, 305, 24, 12517, 633, 3, 93145, 5683, 8351593, 3194, 27, 14992,
               5461306, 10, 5652, 2173, 4, 7046547, 18, 15, 286181, 105, 142572)

_cdf_cache: dict = {}


def zipf(rows: int, n: int, rng, s: float = 1.05) -> np.ndarray:
    key = (rows, s)
    if key not in _cdf_cache:
        p = np.arange(1, rows + 1, dtype=np.float64) ** -s
        c = np.cumsum(p)
        _cdf_cache[key] = c / c[-1]
    return np.minimum(np.searchsorted(_cdf_cache[key], rng.random(n), side="right"), rows - 1).astype(np.int64)


def _time_graph(fn, steps: int, warmup: int = 3) -> float:
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def _dlrm_host_batch(cfg, B, rng, bag_lo, bag_hi):
    dense = rng.standard_normal((B, cfg.n_dense)).astype(np.float32)
    labels = (rng.random(B) < 0.19).astype(np.float64)
    sparse = []
    for rows in cfg.rows_per_field:
        sizes = rng.integers(bag_lo, bag_hi + 1, size=B)
        idx = zipf(rows, int(sizes.sum()), rng)
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        sparse.append((idx, off))
    return dense, sparse, labels


def _dlrm_batch(cfg, B, rng, dev, bag_lo, bag_hi, host=None):
    dense, sparse, labels = host if host is not None else _dlrm_host_batch(cfg, B, rng, bag_lo, bag_hi)
    return (torch.from_numpy(dense).to(dev), [(torch.from_numpy(i).to(dev), torch.from_numpy(o).to(dev))
                                              for i, o in sparse], torch.from_numpy(labels).to(dev))


# ------------------------------------------------------------------ roofline model
def table_counts(idx, off, m3):
    """T, B, P, S, U of one table's batch (the reference's counters)."""
    bag = np.repeat(np.arange(off.size - 1), np.diff(off))
    key = idx // m3
    P = np.unique(key).size
    S = np.unique(bag.astype(np.int64) * (int(key.max()) + 1) + key).size
    return {"T": int(idx.size), "B": int(off.size - 1), "P": int(P), "S": int(S), "U": int(np.unique(idx).size)}


def tt_flops(shape, c):
    """Algorithmic fwd + bwd FLOPs of one TT table step (bench.algorithmic_counts)."""
    import bench
    _, fwd, bwd, nbytes = bench.algorithmic_counts(shape, c["T"], c["B"], c["P"], c["S"], c["U"])
    return fwd + bwd, nbytes


def dlrm_roofline(cfg, host, ms, peak_tflops, hbm_gbs):
    """FP32 roofline of one DLRM training step: the TT fields' algorithmic
    FLOPs (SURVEY.md §8d per field) plus the MLPs' (forward, input and weight
    gradients: 3 x 2 B in out per layer) at the measured FP32 peak."""
    from paper_2507_14668_b200.geometry import TtShape, factorize_dims
    dense, sparse, labels = host
    B = dense.shape[0]
    tt_fl, tt_bytes = 0, 0
    for rows, (idx, off) in zip(cfg.rows_per_field, sparse):
        if rows >= cfg.tt_threshold:
            m, n = factorize_dims(rows, cfg.emb_dim, len(cfg.ranks) - 1)
            shape = TtShape(m, n, cfg.ranks)
            f, nb = tt_flops(shape, table_counts(idx, off, m[-1]))
            tt_fl, tt_bytes = tt_fl + f, tt_bytes + nb
    v = len(cfg.rows_per_field) + 1
    sizes = [(cfg.n_dense, *cfg.bottom_sizes, cfg.emb_dim), (cfg.emb_dim + v * (v - 1) // 2, *cfg.top_sizes, 1)]
    mlp = sum(6 * B * a * b for sz in sizes for a, b in zip(sz[:-1], sz[1:]))
    t = max((tt_fl + mlp) / (peak_tflops * 1e12), tt_bytes / (hbm_gbs * 1e9))
    return {"bound": "fp32", "flops_tt": tt_fl, "flops_mlp": mlp, "peak": peak_tflops, "unit": "TFLOP/s",
            "achieved": (tt_fl + mlp) / (ms * 1e-3) / 1e12, "roofline_ms": t * 1e3, "frac": t * 1e3 / ms,
            "note": "whole step: TT-field fwd+bwd algorithmic FLOPs (SURVEY.md §8d) + MLP 6 B in out, at the "
                    "measured FP32 FMA peak"}


# ------------------------------------------------------------------ CPU baselines (oracle ports, 1 thread)
def _one_thread():
    from threadpoolctl import threadpool_limits
    return threadpool_limits(1)


def cpu_dlrm(cfg, host, budget_s=8.0, max_steps=50):
    """The reference's DLRM train_step (oracle/dlrm_oracle.py restates
    model.py:347-365; pinned bit-exact on the reference's goldens) on this
    host, one thread, on the same synthetic batch shape."""
    import time
    from oracle import dlrm_oracle as D
    dense, sparse, labels = host
    params, fields = D.init_params(cfg.rows_per_field, cfg.emb_dim, cfg.ranks, cfg.tt_threshold, cfg.n_dense,
                                   cfg.bottom_sizes, cfg.top_sizes, seed=0)
    vel, n = {}, 0
    with _one_thread():
        t0 = time.perf_counter()
        while n == 0 or (time.perf_counter() - t0 < budget_s and n < max_steps):
            D.train_step(params, fields, dense, sparse, labels, 0.05, 0.9, vel)
            n += 1
        dt = time.perf_counter() - t0
    B = dense.shape[0]
    return {"value": n * B / dt, "unit": "samples/s", "cores": 1, "kind": "port",
            "sample": f"{n} train steps x {B} samples (oracle/dlrm_oracle.py, fp32 parameters, fp64 gradients), "
                      f"{dt:.1f} s"}


def cpu_table(shape_m, T_bags, pooling, permuted, budget_s=8.0):
    """One config-3 table step of the reference (forward_batch +
    unique_aggregate + tt_core_grads + fused_update: lookup.py:236-296,
    backward.py:72-227 via oracle/ttb_oracle.py), one thread."""
    import time
    from oracle import ttb_oracle as O
    M = 10_000_000
    g = O.Geometry(tuple(shape_m), (4, 4, 4), (1, 32, 32, 1))
    cores = [c.astype(np.float32) for c in O.init_cores(g, 0)]
    rng = np.random.default_rng(5)
    ids = zipf(M, T_bags * pooling, rng)
    if permuted:
        ids = np.random.default_rng(123).permutation(M)[ids]
    off = np.arange(0, T_bags * pooling + 1, pooling, dtype=np.int64)
    gout = (rng.standard_normal((T_bags, 64)) / T_bags).astype(np.float32)
    vel, n = [None] * 3, 0
    with _one_thread():
        t0 = time.perf_counter()
        while n == 0 or time.perf_counter() - t0 < budget_s:
            O.forward(cores, g, ids, off)
            rows, ug = O.unique_aggregate(ids, np.repeat(gout, pooling, axis=0))
            for k, gk in enumerate(O.core_grads(cores, g, rows, ug)):
                vel[k] = O.sgd_step(cores[k], gk, 0.05, 0.9, vel[k])
            n += 1
        dt = time.perf_counter() - t0
    return {"value": n * ids.size / dt, "unit": "lookups/s", "cores": 1, "kind": "port",
            "sample": f"{n} step(s) of one table, {T_bags} bags x pooling {pooling} = {ids.size} lookups "
                      f"({'permuted' if permuted else 'native'} Zipf ids; oracle/ttb_oracle.py), {dt:.1f} s"}


def dlrm_samples_per_s(cfg, B, bag_lo, bag_hi, steps, dev, peaks=None, cpu_B=None):
    from paper_2507_14668_b200.model import DlrmModel
    torch.backends.cuda.matmul.allow_tf32 = False
    rng = np.random.default_rng(11)
    model = DlrmModel(cfg, device=dev, max_indices=B * bag_hi * len(cfg.rows_per_field), check_errors=False,
                      batch_size=B)
    host = _dlrm_host_batch(cfg, B, rng, bag_lo, bag_hi)
    dense, sparse, labels = _dlrm_batch(cfg, B, rng, dev, bag_lo, bag_hi, host=host)
    ms = _time_graph(lambda: model.train_step(dense, sparse, labels, 0.05, 0.9, sync_loss=False), steps)
    ntt = sum(1 for r in cfg.rows_per_field if r >= cfg.tt_threshold)
    res = {"value": B / (ms / 1e3), "unit": "samples/s", "ms_per_step": ms, "batch": B, "tt_fields": ntt,
           "fields": cfg.n_sparse}
    if peaks is not None:
        res["roofline"] = dlrm_roofline(cfg, host, ms, *peaks)
    if cpu_B is not None:
        sub_host = host if cpu_B == B else _dlrm_host_batch(cfg, cpu_B, np.random.default_rng(12), bag_lo, bag_hi)
        res["cpu_baseline"] = cpu_dlrm(cfg, sub_host)
    return res


def cfg1(dev, steps=50, peaks=None, cpu=False):
    from paper_2507_14668_b200.model import ModelConfig
    cfg = ModelConfig(n_dense=6, rows_per_field=(1_000_000,), emb_dim=16, ranks=(1, 16, 16, 1), tt_threshold=1000,
                      bottom_sizes=(64,), top_sizes=(64, 32), loss="bce", seed=0)
    r = dlrm_samples_per_s(cfg, 256, 1, 3, steps, dev, peaks, 256 if cpu else None)
    r["workload"] = "cfg1: DLRM, 1 TT field 1M x 16 ranks 16, bags 1-3 Zipf(1.05), batch 256, SGD momentum 0.9"
    return r


def cfg4(dev, steps=5, B=65536, peaks=None, cpu=False):
    from paper_2507_14668_b200.model import ModelConfig
    cfg = ModelConfig(n_dense=13, rows_per_field=KAGGLE_ROWS, emb_dim=64, ranks=(1, 32, 32, 1), tt_threshold=1000,
                      bottom_sizes=(512, 256), top_sizes=(512, 256), loss="bce", seed=0)
    r = dlrm_samples_per_s(cfg, B, 1, 1, steps, dev, peaks, 2048 if cpu else None)
    r["workload"] = (f"cfg4: Criteo-Kaggle-shaped TT-DLRM, 26 fields (15 TT, tt_threshold 1000), emb 64, ranks 32, "
                     f"bottom 512-256-64, top 512-256-1, batch {B}, fp32 MLPs")
    return r


def cfg5(dev, world=1, rank=0, steps=5, global_batch=524288):
    """BASELINE config 5: the config-4 TT-DLRM trained data parallel — global
    batch 524,288 split over the ranks, one NCCL all-reduce of every gradient
    per step (DlrmModel.train_step_dp); time = max over ranks."""
    import torch.distributed as dist
    from paper_2507_14668_b200.model import DlrmModel, ModelConfig
    torch.backends.cuda.matmul.allow_tf32 = False
    cfg = ModelConfig(n_dense=13, rows_per_field=KAGGLE_ROWS, emb_dim=64, ranks=(1, 32, 32, 1), tt_threshold=1000,
                      bottom_sizes=(512, 256), top_sizes=(512, 256), loss="bce", seed=0)
    B = global_batch // world
    rng = np.random.default_rng(11 + rank)
    model = DlrmModel(cfg, device=dev, max_indices=B * len(cfg.rows_per_field), check_errors=False, batch_size=B)
    dense, sparse, labels = _dlrm_batch(cfg, B, rng, dev, 1, 1)
    step = lambda: model.train_step_dp(dense, sparse, labels, 0.05, 0.9, global_batch=global_batch)  # noqa: E731
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        step()
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"value": global_batch / (ms / 1e3), "unit": "samples/s", "ms_per_step": ms, "global_batch": global_batch,
            "batch_per_gpu": B, "n_gpus": world,
            "workload": f"cfg5: config-4 TT-DLRM, data parallel over {world} GPU(s), global batch {global_batch}, "
                        "one all-reduce of TT-core + dense-field + MLP gradients per step, SGD momentum 0.9, "
                        "fp32 MLPs, eager (not graph-captured)"}


def cfg3(dev, steps=3, B=65536, pooling=20, permuted=False, tables=26, peaks=None, cpu=False):
    from paper_2507_14668_b200.engine import TtEngine
    from paper_2507_14668_b200.geometry import TtShape, factorize_dims, init_random_cores
    M = 10_000_000
    m, n = factorize_dims(M, 64, 3)
    shape = TtShape(m, n, (1, 32, 32, 1))
    T = B * pooling
    eng = TtEngine(shape, T, B, dev)  # one workspace, tables stepped in turn
    rng = np.random.default_rng(3)
    perm = np.random.default_rng(123).permutation(M) if permuted else None
    cores, vel, idxs, host_ids = [], [], [], None
    for t in range(tables):
        cores.append([torch.from_numpy(c).to(dev) for c in init_random_cores(shape, t)])
        vel.append([torch.zeros(c.shape, dtype=torch.float64, device=dev) for c in cores[-1]])
        ids = zipf(M, T, rng)
        if perm is not None:
            ids = perm[ids]
        host_ids = ids
        idxs.append(torch.from_numpy(ids).to(dev))
    off = torch.arange(0, T + 1, pooling, dtype=torch.int64, device=dev)
    gout = torch.randn((B, 64), device=dev) / B  # batch-mean loss scale
    out = torch.empty((B, 64), device=dev)

    def step():
        for t in range(tables):
            eng.plan(idxs[t], off)
            eng.forward(cores[t], out=out)
            eng.backward_sgd(cores[t], gout, 0.05, 0.9, vel[t])

    step()
    torch.cuda.synchronize()
    st = eng.check_errors()
    st.update(eng.plan_counts())  # S and U of the last table's plan, counted on the device
    ms_loop = _time_graph(step, steps, warmup=1)
    del eng
    # the same 26 tables through ONE table-batched handle (§8 f1): one plan /
    # forward / backward + update launch set over all tables' lookups
    from paper_2507_14668_b200.collection import BatchedTtEngine
    beng = BatchedTtEngine([shape] * tables, B, T * tables, dev)
    M = beng.M
    bcores = [torch.zeros(beng.shape.core_extent(k), dtype=torch.float32, device=dev) for k in range(3)]
    for t in range(tables):
        for k in range(3):
            w = shape.m[k] * shape.n[k]
            bcores[k][:, t * M[k] * shape.n[k]: t * M[k] * shape.n[k] + w, :] = cores[t][k]
    bvel = [torch.zeros(c.shape, dtype=torch.float64, device=dev) for c in bcores]
    bidx = torch.cat(idxs)
    boff = torch.arange(0, T * tables + 1, pooling, dtype=torch.int64, device=dev)
    bgout = gout.repeat(tables, 1)
    bout = torch.empty((B * tables, 64), device=dev)
    del cores, vel, idxs, out

    def bstep():
        beng.plan(bidx, boff)
        beng.forward(bcores, out=bout)
        beng.backward_sgd(bcores, bgout, 0.05, 0.9, bvel)

    bstep()
    torch.cuda.synchronize()
    beng.check_errors()
    ms = _time_graph(bstep, steps, warmup=1)
    res = {"value": tables * T / (ms / 1e3), "unit": "lookups/s", "ms_per_step": ms, "tables": tables,
           "lookups_per_table": T, "last_table_counts": {k: st[k] for k in ("P", "S", "U")},
           "per_table_loop": {"ms_per_step": ms_loop, "value": tables * T / (ms_loop / 1e3)},
           "workload": f"cfg3: {tables} TT tables 10M x 64 ranks 32, Zipf(1.05) {'permuted' if permuted else 'native'} "
                       f"ids, pooling {pooling}, {B} bags/table; step = plan+fwd+bwd+SGD of all tables through "
                       "one table-batched handle (per_table_loop: the same, one table at a time)"}
    if peaks is not None:  # per table (the last one's counts; the tables' batches are identically distributed)
        c = table_counts(host_ids, np.arange(0, T + 1, pooling), shape.m[-1])
        fl, nb = tt_flops(shape, c)
        t = max(fl / (peaks[0] * 1e12), nb / (peaks[1] * 1e9)) * tables
        res["roofline"] = {"bound": "fp32", "flops_per_table": fl, "bytes_per_table": nb, "peak": peaks[0],
                           "unit": "TFLOP/s", "achieved": fl * tables / (ms * 1e-3) / 1e12,
                           "roofline_ms": t * 1e3, "frac": t * 1e3 / ms, "counts": c,
                           "note": "SURVEY.md §8d fwd + bwd FLOPs per table at the measured FP32 FMA peak"}
    if cpu:
        res["cpu_baseline"] = cpu_table(shape.m, 4096, pooling, permuted)
    return res


def run_all(dev, peaks=None, cpu=True) -> dict:
    """peaks = (measured FP32 TFLOP/s, HBM GB/s) for the roofline blocks; cpu:
    add the reference's CPU path (oracle ports, one thread) per config."""
    res = {}
    for name, fn in (("cfg1_dlrm", lambda: cfg1(dev, peaks=peaks, cpu=cpu)),
                     ("cfg3_native", lambda: cfg3(dev, peaks=peaks, cpu=cpu)),
                     ("cfg3_permuted", lambda: cfg3(dev, permuted=True, peaks=peaks, cpu=cpu)),
                     ("cfg4_dlrm", lambda: cfg4(dev, peaks=peaks, cpu=cpu))):
        try:
            res[name] = fn()
        except Exception as e:  # report, do not hide: an extra that fails is listed with its error
            res[name] = {"error": f"{type(e).__name__}: {e}"}
        torch.cuda.empty_cache()
    return res
