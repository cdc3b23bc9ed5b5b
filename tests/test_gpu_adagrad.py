"""Adagrad core update (BASELINE north_star item 3: "fused with the
SGD/Adagrad core update") against oracle.adagrad_step — which restates
torch.optim.Adagrad and is pinned against it (test_oracle_golden.py). The
reference has no Adagrad, so this rule's parity to the
reference is unpinned by construction; the gradients feeding it are the
reference's (tt_core_grads, backward.py:101-183)."""
import numpy as np
import pytest
import torch

from oracle import ttb_oracle as O

pytestmark = pytest.mark.gpu


def rel_err(got, want, floor=1e-3):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return float(np.abs(got - want).max() / max(floor, float(np.abs(want).max())))


def batch(rng, rows, B, max_bag):
    sizes = rng.integers(1, max_bag + 1, size=B)
    idx = rng.integers(0, rows, size=int(sizes.sum())).astype(np.int64)
    return idx, np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


@pytest.mark.parametrize("deterministic", [False, True])
def test_fused_adagrad_steps_match_oracle(deterministic):
    from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
    emb = TTEmbeddingBag(10000, 64, (1, 32, 32, 1), tt_m=(20, 20, 25), tt_n=(4, 4, 4), seed=6,
                         deterministic=deterministic)
    emb.enable_fused_adagrad(0.01, eps=1e-10)
    assert emb.engine.fast != deterministic
    g = O.Geometry(emb.shape.m, emb.shape.n, emb.shape.ranks)
    ref = [c.detach().cpu().numpy().astype(np.float32).copy() for c in emb.cores]
    st = [None] * 3
    rng = np.random.default_rng(8)
    for step in range(3):
        idx, off = batch(rng, 10000, 600, 3)
        now = [c.detach().cpu().numpy().astype(np.float64) for c in emb.cores]
        out = emb(torch.from_numpy(idx).cuda(), torch.from_numpy(off[:-1]).cuda())
        # the forward on the cores the GPU holds (the images follow every update)
        assert rel_err(out.detach().cpu().numpy(), O.forward(now, g, idx, off)) < 1e-5, step
        c64 = [c.astype(np.float64) for c in ref]
        gout = rng.standard_normal(out.shape).astype(np.float32)
        out.backward(torch.from_numpy(gout).cuda())
        rows, ug = O.unique_aggregate(idx, np.repeat(gout.astype(np.float64), np.diff(off), axis=0))
        for k, gk in enumerate(O.core_grads(c64, g, rows, ug)):
            st[k] = O.adagrad_step(ref[k], gk, 0.01, 1e-10, st[k])
    for k in range(3):
        # the trajectory: each update inherits the gradients' (1e-4-pinned) error
        assert rel_err(emb.cores[k].detach().cpu().numpy(), ref[k]) < 5e-5, k
        assert rel_err(emb.state_sum[k].cpu().numpy(), st[k]) < 1e-4, k


@pytest.mark.parametrize("deterministic", [False, True])
def test_adagrad_rejects_non_finite_and_leaves_state(deterministic):
    from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
    emb = TTEmbeddingBag(10000, 64, (1, 32, 32, 1), tt_m=(20, 20, 25), tt_n=(4, 4, 4), seed=6,
                         deterministic=deterministic)
    emb.enable_fused_adagrad(0.01)
    rng = np.random.default_rng(9)
    idx, off = batch(rng, 10000, 300, 2)
    before = [c.detach().clone() for c in emb.cores]
    sbefore = [s.clone() for s in emb.state_sum]
    out = emb(torch.from_numpy(idx).cuda(), torch.from_numpy(off[:-1]).cuda())
    gout = torch.randn_like(out)
    gout[7, 3] = float("nan")
    with pytest.raises(ValueError):
        out.backward(gout)
    for c, b in zip(emb.cores, before):
        assert torch.equal(c.detach(), b)
    for s, b in zip(emb.state_sum, sbefore):
        assert torch.equal(s, b)


def test_flat_adagrad_update_bit_exact():
    """ttb_adagrad_update on a flat parameter equals the oracle bit for bit
    (fp64 state via fma, one rounding into fp32), and a latched error word
    cancels it."""
    from paper_2507_14668_b200 import _native as nat
    from paper_2507_14668_b200.engine import _ptr, _stream
    lib = nat.load()
    rng = np.random.default_rng(10)
    n = 100_003
    p = rng.standard_normal(n).astype(np.float32)
    s = rng.random(n)
    g = rng.standard_normal(n).astype(np.float32)
    dp, ds, dg = torch.from_numpy(p.copy()).cuda(), torch.from_numpy(s.copy()).cuda(), torch.from_numpy(g).cuda()
    nat.check(lib.ttb_adagrad_update(_ptr(dp), _ptr(dg), _ptr(ds), n, 0.05, 1e-10, None, _stream()))
    want_s = O.adagrad_step(p, g, 0.05, 1e-10, s.copy())
    assert np.array_equal(dp.cpu().numpy(), p) and np.array_equal(ds.cpu().numpy(), want_s)
    err = torch.ones(1, dtype=torch.int32, device="cuda")
    keep = dp.clone()
    nat.check(lib.ttb_adagrad_update(_ptr(dp), _ptr(dg), _ptr(ds), n, 0.05, 1e-10, _ptr(err), _stream()))
    assert torch.equal(dp, keep)


@pytest.mark.parametrize("deterministic", [False, True])
@pytest.mark.parametrize("pool", [1, 3])
def test_allow_empty_bags_pool_to_zero(deterministic, pool):
    """TTEmbeddingBag(allow_empty_bags=True): empty bags give zero rows and no
    gradient, as torch.nn.EmbeddingBag; the other bags match the oracle
    (which, like the reference, rejects empty bags: it runs on the non-empty
    ones). Default: ValueError (lookup.py:90-91)."""
    from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
    emb = TTEmbeddingBag(10000, 64, (1, 32, 32, 1), tt_m=(20, 20, 25), tt_n=(4, 4, 4), seed=2,
                         deterministic=deterministic, allow_empty_bags=True)
    g = O.Geometry(emb.shape.m, emb.shape.n, emb.shape.ranks)
    rng = np.random.default_rng(11 + pool)
    B = 400
    sizes = rng.integers(1, pool + 1, size=B)
    sizes[rng.random(B) < 0.2] = 0
    sizes[3] = 2  # T = B with empty bags still needs the pooled path
    idx = rng.integers(0, 10000, size=int(sizes.sum())).astype(np.int64)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    out = emb(torch.from_numpy(idx).cuda(), torch.from_numpy(off[:-1]).cuda())
    got = out.detach().cpu().numpy()
    keep = sizes > 0
    c64 = [c.detach().cpu().numpy().astype(np.float64) for c in emb.cores]
    want = O.forward(c64, g, idx, np.concatenate([[0], np.cumsum(sizes[keep])]))
    assert np.array_equal(got[~keep], np.zeros_like(got[~keep]))
    assert rel_err(got[keep], want) < 1e-5
    gout = rng.standard_normal(out.shape).astype(np.float32)
    out.backward(torch.from_numpy(gout).cuda())
    rows, ug = O.unique_aggregate(idx, np.repeat(gout.astype(np.float64), sizes, axis=0))
    for k, gk in enumerate(O.core_grads(c64, g, rows, ug)):
        assert rel_err(emb.cores[k].grad.cpu().numpy(), gk) < 1e-4, k
    strict = TTEmbeddingBag(10000, 64, (1, 32, 32, 1), tt_m=(20, 20, 25), tt_n=(4, 4, 4), seed=2,
                            deterministic=deterministic)
    with pytest.raises(ValueError):
        strict(torch.from_numpy(idx).cuda(), torch.from_numpy(off[:-1]).cuda())
