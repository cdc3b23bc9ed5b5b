"""Generates tests/golden/*.npz by running the UNMODIFIED reference (Rec-AD
artifact, pure numpy) in the build container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference does not exist on the GPU box, so its outputs are frozen here
and committed; tests/test_oracle_golden.py pins the oracle against them and
the GPU parity tests compare the CUDA path against them too.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from ttemb import backward as bw  # noqa: E402
from ttemb import lookup as lk  # noqa: E402
from ttemb import model as md  # noqa: E402
from ttemb import data as dd  # noqa: E402
from ttemb.tt_core import TtShape, TtTable, factorize_dims, init_random, linear_index_to_tt_index  # noqa: E402

OUT = Path(__file__).resolve().parent


def random_table(rng, d, max_rank=8, max_factor=4, dtype=np.float64):
    # same generator shape as the reference tests' fixture (test_tt_core.py:50-56)
    m = tuple(int(rng.integers(1, max_factor + 1)) for _ in range(d))
    n = tuple(int(rng.integers(1, max_factor + 1)) for _ in range(d))
    ranks = (1, *(int(rng.integers(1, max_rank + 1)) for _ in range(d - 1)), 1)
    shape = TtShape(m, n, ranks)
    cores = [rng.standard_normal(shape.core_extent(k)).astype(dtype) for k in range(d)]
    return TtTable(shape, cores)


def pack_table(prefix, table, store):
    store[f"{prefix}.m"] = np.array(table.shape.m)
    store[f"{prefix}.n"] = np.array(table.shape.n)
    store[f"{prefix}.r"] = np.array(table.shape.ranks)
    for k, c in enumerate(table.cores):
        store[f"{prefix}.core{k}"] = c


def batch_arrays(batch):
    idx = np.array([i for bag in batch for i in bag], dtype=np.int64)
    off = np.concatenate([[0], np.cumsum([len(b) for b in batch])]).astype(np.int64)
    return idx, off


def gen_factorize():
    s = {}
    rows_list = list(range(1, 300)) + [1000, 4000, 4096, 100_000, 1_000_000, 2_202_608, 10_000_000, 10_131_227]
    res = []
    for d in (2, 3):
        for r in rows_list:
            m, _ = factorize_dims(r, 4, d)
            res.append([d, r] + m + [0] * (3 - d))
    s["rows"] = np.array(res, dtype=np.int64)
    cols = []
    for d in (2, 3):
        for c in (1, 2, 3, 4, 6, 7, 8, 12, 16, 24, 32, 64, 128):
            try:
                _, n = factorize_dims(100, c, d)
                cols.append([d, c] + n + [0] * (3 - d))
            except ValueError:
                cols.append([d, c, -1, -1, -1])
    s["cols"] = np.array(cols, dtype=np.int64)
    dig = []
    for m in ([2, 3, 2], [4, 4], [10, 10, 10], [1, 5, 3], [200, 200, 250]):
        total = int(np.prod(m))
        for i in sorted(set([0, 1, 5, 15, total - 1] + list(range(0, total, max(1, total // 37))))):
            if i < total:
                dd_ = linear_index_to_tt_index(i, m)
                dig.append([len(m), *m, *([0] * (3 - len(m))), i, *dd_, *([0] * (3 - len(m)))])
    s["digits"] = np.array(dig, dtype=np.int64)
    np.savez_compressed(OUT / "factorize.npz", **s)


def gen_init():
    s = {}
    for j, (rows, dim, ranks, seed) in enumerate([(1000, 16, (1, 8, 8, 1), 0), (4000, 16, (1, 4, 4, 1), 7),
                                                  (500, 8, (1, 3, 1), 3), (1_000_000, 16, (1, 16, 16, 1), 0)]):
        d = len(ranks) - 1
        m, n = factorize_dims(rows, dim, d)
        t = init_random(TtShape(m, n, ranks), seed=seed, dtype=np.float32)
        s[f"c{j}.args"] = np.array([rows, dim, seed, d], dtype=np.int64)
        pack_table(f"c{j}", t, s)
    np.savez_compressed(OUT / "init.npz", **s)


def gen_plans_forward():
    s = {}
    cube = TtTable(TtShape((2, 2, 2), (2, 2, 2), (1, 2, 2, 1)),
                   [np.random.default_rng(0).standard_normal(e) for e in [(1, 4, 2), (2, 4, 2), (2, 4, 1)]])
    frozen = [[1, 0], [7, 2, 3, 0], [5, 5, 5], [4, 1, 4, 6]]
    for j, idx in enumerate(frozen):
        plan = lk.prepare_reuse_plan(idx, cube)
        s[f"frozen{j}.idx"] = np.array(idx)
        s[f"frozen{j}.work"] = np.array(plan.work, dtype=np.int64).reshape(-1, 4)
        s[f"frozen{j}.hits_misses"] = np.array([plan.hits, plan.misses])
    pack_table("cube", cube, s)
    rng = np.random.default_rng(2024)
    cases = 0
    for trial in range(24):
        d = 2 if trial % 4 == 0 else 3
        dtype = np.float32 if trial % 2 else np.float64
        table = random_table(rng, d, dtype=dtype)
        rows = table.shape.rows
        nb = int(rng.integers(1, 9))
        batch = [rng.integers(0, rows, size=int(rng.integers(1, 7))).tolist() for _ in range(nb)]
        idx, off = batch_arrays(batch)
        p = f"case{cases}"
        pack_table(p, table, s)
        s[f"{p}.idx"], s[f"{p}.off"] = idx, off
        out, c = lk.forward_batch(table, batch, use_reuse=True)
        s[f"{p}.out"] = out
        s[f"{p}.counters"] = np.array([c.slice_mults, c.row_adds, c.buffer_hits, c.buffer_misses])
        out_d, cd = lk.forward_batch(table, batch, use_reuse=False)
        s[f"{p}.out_direct"] = out_d
        if d == 3:
            plan = lk.prepare_reuse_plan(idx, table)
            s[f"{p}.work"] = np.array(plan.work, dtype=np.int64).reshape(-1, 4)
            slot_occ = np.array([plan.slot_of[int(k)] for k in (idx // table.shape.m[2])], dtype=np.int64)
            s[f"{p}.slot_occ"] = slot_occ
            bag_ids = np.repeat(np.arange(nb), np.diff(off))
            seg_ids, seg_inv = np.unique(bag_ids * plan.buf_len + slot_occ, return_inverse=True)
            s[f"{p}.seg_ids"], s[f"{p}.seg_inv"] = seg_ids, seg_inv.reshape(-1)
            buf = lk.execute_prefix_products(table, plan)
            s[f"{p}.slots"] = buf.slots
        cases += 1
    s["ncases"] = np.array(cases)
    np.savez_compressed(OUT / "forward.npz", **s)


def gen_backward():
    s = {}
    grads = np.array([[1.0, 0.0], [0.0, 1.0], [2.0, 2.0], [5.0, 5.0]])
    u, g = bw.unique_aggregate([3, 1, 3, 0], grads)
    s["ua_frozen.rows"], s["ua_frozen.grads"] = u, g
    rng = np.random.default_rng(77)
    cases = 0
    for trial in range(16):
        d = 2 if trial % 4 == 0 else 3
        dtype = np.float32 if trial % 2 else np.float64
        table = random_table(rng, d, max_rank=6, max_factor=4, dtype=dtype)
        rows = table.shape.rows
        nb = int(rng.integers(1, 7))
        batch = [rng.integers(0, max(1, rows // 2 + 1), size=int(rng.integers(1, 6))).tolist() for _ in range(nb)]
        idx, off = batch_arrays(batch)
        gout = rng.standard_normal((nb, table.shape.cols)).astype(dtype)
        per_occ = np.repeat(gout, np.diff(off), axis=0)
        uidx, ug = bw.unique_aggregate(idx, per_occ)
        buffer = None
        if d == 3:
            plan = lk.prepare_reuse_plan(idx, table)
            buffer = lk.execute_prefix_products(table, plan)
        cnt = lk.OpCounters()
        cg = bw.tt_core_grads(table, uidx, ug, buffer=buffer, counters=cnt)
        p = f"case{cases}"
        pack_table(p, table, s)
        s[f"{p}.idx"], s[f"{p}.off"], s[f"{p}.gout"] = idx, off, gout
        s[f"{p}.urows"], s[f"{p}.ugrads"] = uidx, ug
        for k, a in enumerate(cg.arrays):
            s[f"{p}.grad{k}"] = a
        s[f"{p}.mults"] = np.array(cnt.slice_mults)
        # fused update: plain SGD then two momentum steps
        for mu in (0.0, 0.9):
            t2 = table.copy()
            opt = bw.OptimizerState(lr=0.05, momentum=mu)
            bw.fused_update(t2, cg, opt)
            bw.fused_update(t2, cg, opt)
            for k, c in enumerate(t2.cores):
                s[f"{p}.upd{int(mu * 10)}.core{k}"] = c
        cases += 1
    s["ncases"] = np.array(cases)
    np.savez_compressed(OUT / "backward.npz", **s)


def gen_dlrm():
    """A tiny DLRM (one TT field + dense fields), fp32, a few SGD+momentum
    steps: parameters after init and after each step, losses."""
    s = {}
    cfg = md.ModelConfig(n_dense=6, rows_per_field=(4000, 500, 118), emb_dim=16, ranks=(1, 4, 4, 1),
                         tt_threshold=1000, bottom_sizes=(32,), top_sizes=(32, 16), loss="bce", seed=5)
    spec = dd.DatasetSpec(n_samples=96, n_dense=6, rows_per_field=(4000, 500, 118), seed=3)
    ds = dd.gen_synthetic(spec)
    model = md.DlrmModel(cfg, dtype=np.float32)
    for name, arr in model.named_params():
        s[f"init.{name}"] = arr.copy()
    s["ckpt_init"] = np.frombuffer(md.checkpoint_bytes(model), dtype=np.uint8)
    s["data.labels"] = ds.labels
    s["data.dense"] = ds.dense
    for f in range(3):
        idx, off = batch_arrays(ds.bags[f])
        s[f"data.idx{f}"], s[f"data.off{f}"] = idx, off
    losses = []
    bs = 32
    for step in range(3):
        sub = ds.select(np.arange(step * bs, (step + 1) * bs))
        losses.append(model.train_step(sub, lr=0.05, momentum=0.9))
        for name, arr in model.named_params():
            s[f"step{step}.{name}"] = arr.copy()
    s["losses"] = np.array(losses)
    s["config"] = np.array([6, 16, 4, 1000, 5])
    s["ckpt_final"] = np.frombuffer(md.checkpoint_bytes(model), dtype=np.uint8)
    np.savez_compressed(OUT / "dlrm.npz", **s)


def gen_dlrm_tc():
    """The production TT geometry inside a DLRM (emb 64, ranks (1, 32, 32, 1),
    n = (4, 4, 4)): the configuration the GPU's tensor-core pipeline runs
    (BASELINE configs 4/5), one 12,000-row TT field + one dense field, bags of
    1-3 indices, 3 SGD+momentum steps, fp32."""
    s = {}
    rows = (12000, 700)
    cfg = md.ModelConfig(n_dense=5, rows_per_field=rows, emb_dim=64, ranks=(1, 32, 32, 1),
                         tt_threshold=1000, bottom_sizes=(32,), top_sizes=(32,), loss="bce", seed=9)
    spec = dd.DatasetSpec(n_samples=192, n_dense=5, rows_per_field=rows, min_bag=1, max_bag=3, seed=4)
    ds = dd.gen_synthetic(spec)
    model = md.DlrmModel(cfg, dtype=np.float32)
    for name, arr in model.named_params():
        s[f"init.{name}"] = arr.copy()
    s["data.labels"] = ds.labels
    s["data.dense"] = ds.dense
    for f in range(len(rows)):
        idx, off = batch_arrays(ds.bags[f])
        s[f"data.idx{f}"], s[f"data.off{f}"] = idx, off
    losses = []
    bs = 64
    for step in range(3):
        sub = ds.select(np.arange(step * bs, (step + 1) * bs))
        losses.append(model.train_step(sub, lr=0.05, momentum=0.9))
        for name, arr in model.named_params():
            s[f"step{step}.{name}"] = arr.copy()
    s["losses"] = np.array(losses)
    np.savez_compressed(OUT / "dlrm_tc.npz", **s)


def gen_reorder():
    """Frequencies, hot rows, communities and the bijection of the reference's
    reorder pipeline on a skewed synthetic trace with planted clusters."""
    from ttemb import reorder as ro
    s = {}
    rng = np.random.default_rng(41)
    table_len = 600
    perm = rng.permutation(table_len)
    batches = []
    for _ in range(80):
        c = int(rng.integers(0, 12))
        members = perm[c * 50:(c + 1) * 50]
        size = int(rng.integers(1, 9))
        b = rng.choice(members, size=size).tolist()
        if rng.random() < 0.3:
            b.append(int(rng.integers(0, 5)))  # hot head
        batches.append(b)
    freq = ro.count_frequencies(batches, table_len)
    graph, hot = ro.build_index_graph(batches, freq, 0.02)
    comm = ro.detect_communities(graph)
    bij = ro.build_bijection(comm, hot, freq, table_len)
    idx, off = batch_arrays(batches)
    s["idx"], s["off"] = idx, off
    s["table_len"] = np.array([table_len])
    s["counts"], s["row_of_rank"], s["rank_of"] = freq.counts, freq.row_of_rank, freq.rank_of
    s["hot"] = np.array(sorted(hot), dtype=np.int64)
    s["community_of"] = comm.community_of.astype(np.int64)
    s["forward"], s["inverse"] = bij.forward, bij.inverse
    rel = ro.apply_bijection(bij, batches)
    s["relabeled"] = np.concatenate([np.asarray(b, dtype=np.int64) for b in rel])
    s["mdp_before"] = np.array([ro.mean_distinct_prefixes(batches, 8)])
    s["mdp_after"] = np.array([ro.mean_distinct_prefixes(rel, 8)])
    np.savez_compressed(OUT / "reorder.npz", **s)


if __name__ == "__main__":
    gen_factorize()
    gen_init()
    gen_plans_forward()
    gen_backward()
    gen_dlrm()
    gen_dlrm_tc()
    gen_reorder()
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)
