"""The DEFAULT (tensor-core) pipeline pinned on the fp64 oracle at BASELINE
sizes, its own plan checked structurally and bit-exactly, and the error
semantics of the update (B200).

Bars (BASELINE.json north_star): forward within 1e-5 and core gradients
within 1e-4 scale-relative per core against the oracle evaluated in fp64 on
the same fp32 cores; integer plan structures bit-exact against numpy.
Reference functions: forward_batch lookup.py:236-296, tt_core_grads
backward.py:101-183, prepare_reuse_plan lookup.py:97-124, fused_update
backward.py:186-204."""
import numpy as np
import pytest
import torch

from oracle import ttb_oracle as O

pytestmark = pytest.mark.gpu

FWD_TOL = 1e-5
GRAD_TOL = 1e-4
ITEM_LEN, TILE_ITEMS, SORT_ITEMS = 32, 32, 256  # ttb_fast.cuh kItemLen, kTileItems, kSortItems


def rel_err(got, want, floor=1e-3):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    return float(np.abs(got - want).max() / max(floor, float(np.abs(want).max())))


def oracle_grads_chunked(c64, g, idx, off, gout, chunk=8192):
    """tt_core_grads of the aggregated rows, in row chunks (core gradients
    are additive over rows; bounds the oracle's (U, r, n, r) fp64 blocks)."""
    ur, ug = O.unique_aggregate(idx, np.repeat(gout.astype(np.float64), np.diff(off), axis=0))
    acc = None
    for s in range(0, ur.size, chunk):
        part = O.core_grads(c64, g, ur[s:s + chunk], ug[s:s + chunk])
        acc = part if acc is None else [a + b for a, b in zip(acc, part)]
    return acc


def module(rows, seed, T, B, **kw):
    from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
    emb = TTEmbeddingBag(rows, 64, (1, 32, 32, 1), seed=seed, max_indices=T, max_bags=B, **kw)
    assert emb.engine.fast, "these tests pin the tensor-core pipeline"
    return emb


def run_fast(emb, idx, off, gout):
    cores = [c.detach() for c in emb.cores]
    ti, to, tg = torch.from_numpy(idx).cuda(), torch.from_numpy(off).cuda(), torch.from_numpy(gout).cuda()
    emb.engine.plan(ti, to)
    out = emb.engine.forward(cores).cpu().numpy()
    grads = [x.cpu().numpy() for x in emb.engine.backward(cores, tg)]
    emb.engine.check_errors()
    return out, grads, [c.cpu().numpy().astype(np.float64) for c in cores]


def zipf_ids(rows, n, seed, permuted):
    from bench_extras import zipf
    idx = zipf(rows, n, np.random.default_rng(seed))
    if permuted:
        idx = np.random.default_rng(123).permutation(rows)[idx]
    return idx


# ------------------------------------------------------------------ BASELINE sizes vs the oracle
def test_config2_full_batch_vs_oracle():
    """BASELINE configs[1] exactly: 10M x 64, ranks 32, 65,536 bags of one
    uniform index; every pooled row and all three core gradients vs fp64."""
    B = 65_536
    emb = module(10_000_000, 0, B, B)
    g = O.Geometry(emb.shape.m, emb.shape.n, emb.shape.ranks)
    idx = np.random.default_rng(1).integers(0, 10_000_000, B)
    off = np.arange(B + 1, dtype=np.int64)
    gout = np.random.default_rng(2).standard_normal((B, 64)).astype(np.float32)
    out, grads, c64 = run_fast(emb, idx, off, gout)
    assert rel_err(out, O.forward(c64, g, idx, off)) < FWD_TOL
    want = oracle_grads_chunked(c64, g, idx, off, gout)
    for k in range(3):
        assert rel_err(grads[k], want[k]) < GRAD_TOL, k


@pytest.mark.parametrize("permuted", [False, True])
def test_config3_table_vs_oracle(permuted):
    """One BASELINE configs[2] table at the CPU-reference batch:
    B = 4,096 bags of 20 Zipf(1.05) indices, native and permuted ids (hot
    prefixes split into many full work items, repeated rows inside items)."""
    B, pool = 4096, 20
    emb = module(10_000_000, 0, B * pool, B)
    g = O.Geometry(emb.shape.m, emb.shape.n, emb.shape.ranks)
    idx = zipf_ids(10_000_000, B * pool, 4 + permuted, permuted)
    off = np.arange(0, B * pool + 1, pool, dtype=np.int64)
    gout = (np.random.default_rng(7).standard_normal((B, 64)) / B).astype(np.float32)
    out, grads, c64 = run_fast(emb, idx, off, gout)
    assert rel_err(out, O.forward(c64, g, idx, off)) < FWD_TOL
    want = oracle_grads_chunked(c64, g, idx, off, gout)
    for k in range(3):
        assert rel_err(grads[k], want[k]) < GRAD_TOL, (permuted, k)


def test_kaggle_m3_261_field_vs_oracle():
    """The Criteo-Kaggle 10,131,227-row field (m = (171, 227, 261)): G3 just
    fits the forward's shared memory; full forward and gradients vs fp64."""
    T = 8192
    emb = module(10_131_227, 1, T, T)
    assert tuple(emb.shape.m) == (171, 227, 261)
    g = O.Geometry(emb.shape.m, emb.shape.n, emb.shape.ranks)
    rng = np.random.default_rng(14)
    idx = rng.integers(0, 10_131_227, T)
    off = np.arange(T + 1, dtype=np.int64)
    gout = rng.standard_normal((T, 64)).astype(np.float32)
    out, grads, c64 = run_fast(emb, idx, off, gout)
    assert rel_err(out, O.forward(c64, g, idx, off)) < FWD_TOL
    want = oracle_grads_chunked(c64, g, idx, off, gout)
    for k in range(3):
        assert rel_err(grads[k], want[k]) < GRAD_TOL, k


# ------------------------------------------------------------------ k_fplan, bit-exact structure
def _plan_cases():
    rng = np.random.default_rng(31)
    yield "uniform_pool1", 10_000_000, rng.integers(0, 10_000_000, 65_536), 1
    yield "zipf_pool20", 10_000_000, zipf_ids(10_000_000, 4096 * 20, 5, False), 20
    yield "zipf_perm_pool20", 10_000_000, zipf_ids(10_000_000, 4096 * 20, 6, True), 20
    yield "one_hot_row", 10_000_000, np.full(3000, 1234567, dtype=np.int64), 3
    yield "ragged_small", 10_000, None, None


@pytest.mark.parametrize("case", list(range(5)))
def test_fast_plan_structure_bit_exact(case):
    """k_fplan's items, tiles and (bag, i3) list: the multiset of
    (bag, row) over all positions equals the input's; each item holds 1-32
    lookups of ONE prefix; a prefix of c lookups has ceil(c / 32) items; each
    tile holds 1-32 items of one i2, tiles cover the items in order; the CTA
    ranges cover the tiles; P = numpy's distinct prefixes."""
    name, rows, idx, pool = list(_plan_cases())[case]
    if idx is None:  # ragged bags 1..9
        rng = np.random.default_rng(8)
        sizes = rng.integers(1, 10, 700)
        idx = rng.integers(0, rows, int(sizes.sum()))
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        emb = module(rows, 2, idx.size, sizes.size, tt_m=(20, 20, 25), tt_n=(4, 4, 4))
    else:
        off = np.arange(0, idx.size + 1, pool, dtype=np.int64)
        emb = module(rows, 0, idx.size, off.size - 1)
    m1, m2, m3 = emb.shape.m
    eng = emb.engine
    eng.plan(torch.from_numpy(idx).cuda(), torch.from_numpy(off).cuda())
    st = eng.check_errors()
    fp = eng.export_fast_plan()
    T, items, tiles = idx.size, fp["items"], fp["tiles"]
    assert fp["T"] == T
    start, key, sbi = fp["item_start"].astype(np.int64), fp["item_key"].astype(np.int64), fp["sbi"]
    # items: contiguous position runs of 1..32
    assert start[0] == 0 and start[items] == T
    lens = np.diff(start)
    assert lens.min() >= 1 and lens.max() <= ITEM_LEN, name
    # positions -> (bag, row) from the item key (i2-major: key = i2 m1 + i1) and i3
    pos_key = np.repeat(key, lens)
    i1, i2 = pos_key % m1, pos_key // m1
    rows_got = (i1 * m2 + i2) * m3 + sbi[:, 1].astype(np.int64)
    bag_in = np.repeat(np.arange(off.size - 1), np.diff(off))
    got = np.sort(sbi[:, 0].astype(np.int64) * (m1 * m2 * m3) + rows_got)
    want = np.sort(bag_in * (m1 * m2 * m3) + idx)
    assert np.array_equal(got, want), name
    # items per prefix = ceil(count / 32); P
    pk_in = (idx // (m2 * m3)) + m1 * ((idx // m3) % m2)  # i1 + m1 i2
    uk, cnt = np.unique(pk_in, return_counts=True)
    ik, icnt = np.unique(key, return_counts=True)
    assert np.array_equal(uk, ik), name
    assert np.array_equal(icnt, (cnt + ITEM_LEN - 1) // ITEM_LEN), name
    assert st["P"] == uk.size
    # tiles: (i2, first item, n items, first position), in item order, one i2 each
    ti = fp["tile_info"].astype(np.int64)
    assert ti[0, 1] == 0 and np.array_equal(ti[1:, 1], ti[:-1, 1] + ti[:-1, 2]) and ti[-1, 1] + ti[-1, 2] == items
    assert ti[:, 2].min() >= 1 and ti[:, 2].max() <= TILE_ITEMS
    assert np.array_equal(ti[:, 3], start[ti[:, 1]])
    tile_of_item = np.repeat(np.arange(tiles), ti[:, 2])
    assert np.array_equal(key // m1, ti[tile_of_item, 0]), name
    assert np.all(np.diff(ti[:, 0]) >= 0)  # tiles grouped by i2
    # CTA ranges
    cta = fp["cta_tiles"].astype(np.int64)
    assert cta[0] == 0 and cta[-1] == tiles and np.all(np.diff(cta) >= 0)
    # pooled batches (k_rowsort): a prefix with >= 2 full items has them on
    # contiguous positions, sorted by i3 inside each run of SORT_ITEMS items
    if idx.size > off.size - 1:
        i3 = sbi[:, 1].astype(np.int64)
        full = lens == ITEM_LEN
        for k in ik[icnt >= 2]:
            fi = np.nonzero((key == k) & full)[0]
            if fi.size < 2:
                continue
            p0 = start[fi[0]]
            assert np.array_equal(start[fi], p0 + ITEM_LEN * np.arange(fi.size)), (name, k)
            for c in range(0, fi.size, SORT_ITEMS):
                seg = i3[p0 + c * ITEM_LEN: p0 + min(fi.size, c + SORT_ITEMS) * ITEM_LEN]
                assert np.all(np.diff(seg) >= 0), (name, k, c)


@pytest.mark.parametrize("pool,permuted", [(1, False), (20, False), (20, True)])
def test_device_counters_S_U(pool, permuted):
    """S (bag-prefix segments, lookup.py:280-284) and U (distinct rows,
    backward.py:81-87) counted on the device equal numpy's."""
    B = 8192 if pool > 1 else 65_536
    emb = module(10_000_000, 0, B * pool, B)
    m3 = emb.shape.m[2]
    idx = zipf_ids(10_000_000, B * pool, 9, permuted) if pool > 1 else \
        np.random.default_rng(3).integers(0, 10_000_000, B)
    off = np.arange(0, B * pool + 1, pool, dtype=np.int64)
    emb.engine.plan(torch.from_numpy(idx).cuda(), torch.from_numpy(off).cuda())
    c = emb.engine.plan_counts()
    bag = np.repeat(np.arange(B), pool)
    assert c["U"] == np.unique(idx).size
    assert c["S"] == np.unique(bag * (10_000_000 // m3 + 1) + idx // m3).size
    st = emb.engine.status()
    assert st["S"] == c["S"] and st["U"] == c["U"]


def test_device_counters_long_ragged_bags():
    emb = module(10_000, 0, 5000, 64, tt_m=(20, 20, 25), tt_n=(4, 4, 4))
    rng = np.random.default_rng(2)
    sizes = rng.integers(1, 150, 40)
    idx = rng.integers(0, 400, int(sizes.sum())) * 25 + rng.integers(0, 3, int(sizes.sum()))
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    emb.engine.plan(torch.from_numpy(idx).cuda(), torch.from_numpy(off).cuda())
    c = emb.engine.plan_counts()
    bag = np.repeat(np.arange(sizes.size), sizes)
    assert c["U"] == np.unique(idx).size
    assert c["S"] == np.unique(bag * 1000 + idx // 25).size


# ------------------------------------------------------------------ update error semantics
@pytest.mark.parametrize("deterministic", [False, True])
def test_fused_sgd_nonfinite_leaves_cores_untouched(deterministic):
    """fused_update validates every gradient before touching any core
    (backward.py:190-194): a NaN upstream gradient with fused SGD(+momentum)
    raises ValueError and leaves cores AND velocities bitwise unchanged; the
    next good step still matches the oracle."""
    from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
    emb = TTEmbeddingBag(10000, 64, (1, 32, 32, 1), tt_m=(20, 20, 25), tt_n=(4, 4, 4), seed=3,
                         deterministic=deterministic)
    assert emb.engine.fast != deterministic
    emb.enable_fused_sgd(0.05, 0.9)
    rng = np.random.default_rng(5)
    idx = torch.from_numpy(rng.integers(0, 10000, 600)).cuda()
    off = torch.arange(0, 600, 3, device="cuda")
    out = emb(idx, off)
    out.backward(torch.randn_like(out))  # a good step: velocity != 0
    cores0 = [c.detach().clone() for c in emb.cores]
    vel0 = [v.clone() for v in emb.velocity]
    out = emb(idx, off)
    gbad = torch.randn_like(out)
    gbad[7, 3] = float("nan")
    with pytest.raises(ValueError):
        out.backward(gbad)
    for k in range(3):
        assert torch.equal(emb.cores[k].detach(), cores0[k]), k
        assert torch.equal(emb.velocity[k], vel0[k]), k
    # an inf that only appears after accumulation-free products: same
    out = emb(idx, off)
    ginf = torch.zeros_like(out)
    ginf[0, 0] = float("inf")
    with pytest.raises(ValueError):
        out.backward(ginf)
    for k in range(3):
        assert torch.equal(emb.cores[k].detach(), cores0[k]), k
    # the cached core images were rebuilt from the unchanged cores
    out = emb(idx, off)
    g = O.Geometry(emb.shape.m, emb.shape.n, emb.shape.ranks)
    c64 = [c.cpu().numpy().astype(np.float64) for c in cores0]
    offn = np.concatenate([off.cpu().numpy(), [600]])
    assert rel_err(out.detach().cpu().numpy(), O.forward(c64, g, idx.cpu().numpy(), offn)) < FWD_TOL


def test_sgd_update_checked_rejects_nonfinite():
    from paper_2507_14668_b200 import dp
    p = torch.randn(1000, device="cuda")
    v = torch.randn(1000, dtype=torch.float64, device="cuda")
    g = torch.randn(1000, device="cuda")
    g[500] = float("inf")
    p0, v0 = p.clone(), v.clone()
    with pytest.raises(ValueError):
        dp.checked_update(p, g, v, 0.1, 0.9)
    assert torch.equal(p, p0) and torch.equal(v, v0)
    g[500] = 1.0
    dp.checked_update(p, g, v, 0.1, 0.9)
    want_v = v0 * 0.9 + g.double()
    assert torch.equal(v, want_v)
    assert torch.equal(p, (p0.double() - 0.1 * want_v).float())


def test_ops_fused_update_all_or_nothing():
    """ops.fused_update checks all three core gradients before updating any."""
    from paper_2507_14668_b200 import ops
    g = O.Geometry((20, 20, 25), (4, 4, 4), (1, 32, 32, 1))
    cores = [c.astype(np.float32) for c in O.init_cores(g, 1)]
    from paper_2507_14668_b200.geometry import TtShape
    table = ops.GpuTtTable(TtShape(g.m, g.n, g.r), cores)
    before = [c.clone() for c in table.cores]
    grads = [np.ones_like(c) for c in cores]
    grads[2][0, 0, 0] = np.nan  # only the LAST core's gradient is bad
    with pytest.raises(ValueError):
        ops.fused_update(table, ops.CoreGrads(grads), ops.OptimizerState(0.1, 0.5))
    for k in range(3):
        assert torch.equal(table.cores[k], before[k]), k


def test_indices_on_wrong_device_raise():
    from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
    emb = TTEmbeddingBag(10000, 64, (1, 32, 32, 1), tt_m=(20, 20, 25), tt_n=(4, 4, 4))
    with pytest.raises(ValueError):
        emb(torch.tensor([1, 2, 3]), torch.tensor([0, 1]))
    with pytest.raises(ValueError):
        emb(torch.tensor([1, 2, 3], device="cuda"), torch.tensor([0, 1]))


def test_dense_field_empty_and_multi_index_bags():
    """A dense (below tt_threshold) field with as many indices as bags but
    an empty bag next to a two-index bag pools by bag id (model.py:222-226)."""
    from paper_2507_14668_b200.model import DenseField
    f = DenseField(50, 8, seed=1, device="cuda")
    idx = torch.tensor([3, 7], device="cuda")
    off = torch.tensor([0, 2, 2], device="cuda")
    out = f(idx, off)
    rows = f.rows.detach()
    assert torch.allclose(out[0], rows[3] + rows[7]) and torch.equal(out[1], torch.zeros_like(out[1]))


def test_sgd_update_multi_matches_single_updates():
    """ttb_sgd_update_multi (DlrmModel's one-launch update of every non-core
    parameter) is bitwise `count` ttb_sgd_update calls, with and without
    momentum, across more tensors than one launch holds (32)."""
    import ctypes as C
    from paper_2507_14668_b200 import _native as nat
    from paper_2507_14668_b200.engine import _ptr, _stream
    lib = nat.load()
    torch.manual_seed(0)
    sizes = [1, 3, 64, 1000, 17] * 8  # 40 tensors
    for mu in (0.0, 0.9):
        ps = [torch.randn(n, device="cuda") for n in sizes]
        gs = [torch.randn(n, device="cuda") for n in sizes]
        vs = [torch.randn(n, device="cuda", dtype=torch.float64) for n in sizes]
        p1, v1 = [p.clone() for p in ps], [v.clone() for v in vs]
        for p, g, v in zip(p1, gs, v1):
            nat.check(lib.ttb_sgd_update(_ptr(p), _ptr(g), _ptr(v), p.numel(), 0.05, mu, _stream()))
        arr = (nat.TtbSgdTensor * len(sizes))(*[nat.TtbSgdTensor(p.data_ptr(), g.data_ptr(), v.data_ptr(), p.numel())
                                                for p, g, v in zip(ps, gs, vs)])
        nat.check(lib.ttb_sgd_update_multi(arr, len(sizes), 0.05, mu, _stream()))
        torch.cuda.synchronize()
        for a, b in zip(ps, p1):
            assert torch.equal(a, b)
        if mu > 0:
            for a, b in zip(vs, v1):
                assert torch.equal(a, b)
    with pytest.raises(ValueError):
        nat.check(lib.ttb_sgd_update_multi(arr, len(sizes), -1.0, 0.9, _stream()))


# ------------------------------------------------------------------ plan / backward state across calls
def test_plans_of_different_grid_sizes_and_repeated_backward():
    """The plan clears its own header words and the backward's flat gradient
    buffer (no memset nodes), and its grid barrier words are reset by the
    last CTA out: plans whose grids differ (T = 65,536 / 1,500 / 65,536
    pooled) must each give the oracle's forward and gradients, and a second
    backward on the same plan must not see the first one's gradients."""
    rows = 10_000_000
    emb = module(rows, 3, 65_536 * 2, 65_536)
    g = O.Geometry(emb.shape.m, emb.shape.n, emb.shape.ranks)
    rng = np.random.default_rng(41)
    cases = [(rng.integers(0, rows, 65_536), 1), (rng.integers(0, rows, 1_500), 1),
             (zipf_ids(rows, 65_536 * 2, 9, False), 2)]
    for idx, pool in cases:
        off = np.arange(0, idx.size + 1, pool, dtype=np.int64)
        gout = rng.standard_normal((off.size - 1, 64)).astype(np.float32)
        out, grads, c64 = run_fast(emb, idx, off, gout)
        assert rel_err(out, O.forward(c64, g, idx, off)) < FWD_TOL, (idx.size, pool)
        want = oracle_grads_chunked(c64, g, idx, off, gout)
        for k in range(3):
            assert rel_err(grads[k], want[k]) < GRAD_TOL, (idx.size, pool, k)
        # the same plan again: fresh gradients, not accumulated onto the first
        again = [x.cpu().numpy() for x in emb.engine.backward([c.detach() for c in emb.cores],
                                                               torch.from_numpy(gout).cuda())]
        for k in range(3):
            assert np.array_equal(again[k], grads[k]) or rel_err(again[k], want[k]) < GRAD_TOL, (idx.size, k)
        emb.engine.check_errors()
