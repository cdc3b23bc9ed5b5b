"""Table-batched multi-field op: TTEmbeddingBagCollection
runs every table's plan / forward / backward / update in one launch set over
stacked cores. Each table is checked against the oracle for that table alone
(the reference's per-field loop, model.py:295-298 / 334-338): forward within
1e-5, core gradients within 1e-4 (scale-relative), padded core regions
exactly zero."""
import numpy as np
import pytest
import torch

from oracle import ttb_oracle as O

pytestmark = pytest.mark.gpu


def rel_err(got, want, floor=1e-3):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return float(np.abs(got - want).max() / max(floor, float(np.abs(want).max())))


def make_batch(rng, rows_list, B, max_bag, zipf=False):
    idx, sizes = [], []
    for rows in rows_list:
        s = rng.integers(1, max_bag + 1, size=B)
        if zipf:
            p = 1.0 / np.arange(1, rows + 1) ** 1.05
            ids = rng.choice(rows, size=int(s.sum()), p=p / p.sum())
        else:
            ids = rng.integers(0, rows, size=int(s.sum()))
        idx.append(ids.astype(np.int64))
        sizes.append(s)
    allsizes = np.concatenate(sizes)
    off = np.concatenate([[0], np.cumsum(allsizes)]).astype(np.int64)
    return idx, sizes, np.concatenate(idx), off


def per_table(emb, f):
    g = O.Geometry(emb.shapes[f].m, emb.shapes[f].n, emb.shapes[f].ranks)
    return g, [c.detach().cpu().numpy().astype(np.float64) for c in emb.table_cores(f)]


@pytest.mark.parametrize("rows,B,max_bag,zipf", [
    ((10_000, 31_000, 4_000), 300, 1, False),        # one lookup per bag, three different factorisations
    ((10_000, 31_000, 4_000, 77_777), 257, 6, True),  # pooled, skewed
    ((1460, 12517, 93145, 5683), 512, 1, True),       # Criteo-Kaggle TT fields
])
def test_collection_matches_per_table_oracle(rows, B, max_bag, zipf):
    from paper_2507_14668_b200.collection import TTEmbeddingBagCollection
    from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
    emb = TTEmbeddingBagCollection([(r, 64) for r in rows], seeds=[3 + f for f in range(len(rows))],
                                   bags_per_table=B, max_indices=1 << 14)
    rng = np.random.default_rng(len(rows) + B)
    idx, sizes, flat, off = make_batch(rng, rows, B, max_bag, zipf)
    out = emb(torch.from_numpy(flat).cuda(), torch.from_numpy(off[:-1]).cuda())
    assert out.shape == (len(rows), B, 64)
    gout = rng.standard_normal(out.shape).astype(np.float32)
    out.backward(torch.from_numpy(gout).cuda())
    M = emb.engine.M
    for f, r in enumerate(rows):
        # the table's values are a stand-alone TTEmbeddingBag's (same factorisation and init)
        solo = TTEmbeddingBag(r, 64, (1, 32, 32, 1), seed=3 + f)
        for a, b in zip(emb.table_cores(f), solo.cores):
            assert torch.equal(a.detach(), b.detach())
        g, c64 = per_table(emb, f)
        o = np.concatenate([[0], np.cumsum(sizes[f])])
        assert rel_err(out[f].detach().cpu().numpy(), O.forward(c64, g, idx[f], o)) < 1e-5, f
        urows, ug = O.unique_aggregate(idx[f], np.repeat(gout[f].astype(np.float64), sizes[f], axis=0))
        want = O.core_grads(c64, g, urows, ug)
        sh = emb.shapes[f]
        for k in range(3):
            gk = emb.cores[k].grad[:, f * M[k] * 4: f * M[k] * 4 + sh.m[k] * 4, :].cpu().numpy()
            assert rel_err(gk, want[k]) < 1e-4, (f, k)
            pad = emb.cores[k].grad[:, f * M[k] * 4 + sh.m[k] * 4: (f + 1) * M[k] * 4, :]
            assert not pad.any(), (f, k)


def test_collection_fused_sgd_steps():
    from paper_2507_14668_b200.collection import TTEmbeddingBagCollection
    rows = (20_000, 9_000)
    emb = TTEmbeddingBagCollection([(r, 64) for r in rows], seeds=[1, 2], bags_per_table=400)
    emb.enable_fused_sgd(0.05, 0.9)
    refs = [[c.astype(np.float32).copy() for c in per_table(emb, f)[1]] for f in range(2)]
    geoms = [per_table(emb, f)[0] for f in range(2)]
    vel = [[None] * 3 for _ in range(2)]
    rng = np.random.default_rng(7)
    for step in range(3):
        idx, sizes, flat, off = make_batch(rng, rows, 400, 3, zipf=True)
        out = emb(torch.from_numpy(flat).cuda(), torch.from_numpy(off[:-1]).cuda())
        gout = rng.standard_normal(out.shape).astype(np.float32) / 400
        out.backward(torch.from_numpy(gout).cuda())
        for f in range(2):
            c64 = [c.astype(np.float64) for c in refs[f]]
            u, ug = O.unique_aggregate(idx[f], np.repeat(gout[f].astype(np.float64), sizes[f], axis=0))
            for k, gk in enumerate(O.core_grads(c64, geoms[f], u, ug)):
                vel[f][k] = O.sgd_step(refs[f][k], gk, 0.05, 0.9, vel[f][k])
    for f in range(2):
        for k, c in enumerate(emb.table_cores(f)):
            assert rel_err(c.detach().cpu().numpy(), refs[f][k]) < 1e-5, (f, k)


def test_collection_rejects_bad_batches():
    from paper_2507_14668_b200.collection import TTEmbeddingBagCollection
    emb = TTEmbeddingBagCollection([(5000, 64), (6000, 64)], bags_per_table=10)
    idx = torch.arange(20, device="cuda")
    with pytest.raises(ValueError):  # wrong bag count
        emb(idx, torch.arange(0, 18, device="cuda"))
    bad = idx.clone()
    bad[15] = 6000  # table 1 has 6000 rows (its padded rows may be more; factorize_dims pads)
    bad[15] = emb.shapes[1].rows
    with pytest.raises(ValueError):
        emb(bad, torch.arange(0, 20, device="cuda"))
    with pytest.raises(ValueError):  # not the tensor-core geometry
        TTEmbeddingBagCollection([(5000, 16), (6000, 16)], tt_ranks=(1, 16, 16, 1))
