"""CUDA path vs the oracle and the reference's golden vectors (B200).

Bars (BASELINE.json north_star): plan / digits / segments / unique rows
bit-exact; forward within 1e-5 scale-relative (the reference's own metric,
test_lookup.py:176-177); core gradients within 1e-4 scale-relative per core.
Ground truth: the oracle evaluated in fp64 on the fp32 cores."""
import numpy as np
import pytest
import torch

from oracle import ttb_oracle as O

pytestmark = pytest.mark.gpu

FWD_TOL = 1e-5
GRAD_TOL = 1e-4


def rel_err(got, want, floor=1e-3):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    return float(np.abs(got - want).max() / max(floor, float(np.abs(want).max())))


def golden_geom(s, p):
    return O.Geometry(tuple(int(v) for v in s[f"{p}.m"]), tuple(int(v) for v in s[f"{p}.n"]),
                      tuple(int(v) for v in s[f"{p}.r"]))


def make_engine(g, T, B, deterministic=False):
    from paper_2507_14668_b200.engine import TtEngine
    from paper_2507_14668_b200.geometry import TtShape
    return TtEngine(TtShape(g.m, g.n, g.r), max(T, 16), max(B, 16), "cuda", deterministic=deterministic)


def to_dev(cores32):
    return [torch.from_numpy(np.ascontiguousarray(c, dtype=np.float32)).cuda() for c in cores32]


def run_case(g, cores32, idx, off, gout=None, deterministic=False):
    eng = make_engine(g, idx.size, off.size - 1, deterministic)
    dc = to_dev(cores32)
    eng.plan(torch.from_numpy(idx).cuda(), torch.from_numpy(off).cuda())
    out = eng.forward(dc).cpu().numpy()
    res = dict(out=out, eng=eng, dc=dc)
    if gout is not None:
        grads = eng.backward(dc, torch.from_numpy(gout.astype(np.float32)).cuda())
        res["grads"] = [x.cpu().numpy() for x in grads]
    return res


# ------------------------------------------------------------------ golden
def test_plan_bit_exact_golden(golden):
    s = golden("forward")
    ncheck = 0
    for c in range(int(s["ncases"])):
        p = f"case{c}"
        g = golden_geom(s, p)
        if g.d != 3:
            continue
        cores32 = [s[f"{p}.core{k}"].astype(np.float32) for k in range(3)]
        r = run_case(g, cores32, s[f"{p}.idx"], s[f"{p}.off"])
        ex = r["eng"].export_plan()
        assert np.array_equal(ex["work"], s[f"{p}.work"]), p
        assert np.array_equal(ex["slot_occ"], s[f"{p}.slot_occ"]), p
        assert np.array_equal(ex["seg_ids"], s[f"{p}.seg_ids"]), p
        assert np.array_equal(ex["seg_inv"], s[f"{p}.seg_inv"]), p
        digits = np.stack(O.digits_of(s[f"{p}.idx"], g.m), axis=1)
        assert np.array_equal(ex["digits"], digits)
        ncheck += 1
    assert ncheck >= 10


def test_plan_frozen_known_answers(golden):
    s = golden("forward")
    g = O.Geometry((2, 2, 2), (2, 2, 2), (1, 2, 2, 1))
    cores32 = [s[f"cube.core{k}"].astype(np.float32) for k in range(3)]
    for j in range(4):
        idx = s[f"frozen{j}.idx"].astype(np.int64)
        off = np.array([0, idx.size], dtype=np.int64)
        r = run_case(g, cores32, idx, off)
        ex = r["eng"].export_plan()
        assert np.array_equal(ex["work"], s[f"frozen{j}.work"])
        hits, misses = s[f"frozen{j}.hits_misses"]
        assert ex["P"] == misses and ex["T"] - ex["P"] == hits


def test_forward_golden(golden):
    s = golden("forward")
    for c in range(int(s["ncases"])):
        p = f"case{c}"
        g = golden_geom(s, p)
        cores32 = [s[f"{p}.core{k}"].astype(np.float32) for k in range(g.d)]
        r = run_case(g, cores32, s[f"{p}.idx"], s[f"{p}.off"])
        want = O.forward([x.astype(np.float64) for x in cores32], g, s[f"{p}.idx"], s[f"{p}.off"])
        assert rel_err(r["out"], want) < FWD_TOL, p
        if s[f"{p}.core0"].dtype == np.float32:  # the reference's own fp32 output
            assert rel_err(r["out"], s[f"{p}.out"]) < FWD_TOL, p


def test_backward_golden(golden):
    s = golden("backward")
    for c in range(int(s["ncases"])):
        p = f"case{c}"
        g = golden_geom(s, p)
        cores32 = [s[f"{p}.core{k}"].astype(np.float32) for k in range(g.d)]
        idx, off, gout = s[f"{p}.idx"], s[f"{p}.off"], s[f"{p}.gout"].astype(np.float32)
        r = run_case(g, cores32, idx, off, gout)
        per = np.repeat(gout.astype(np.float64), np.diff(off), axis=0)
        ur, ug = O.unique_aggregate(idx, per)
        want = O.core_grads([x.astype(np.float64) for x in cores32], g, ur, ug)
        for k in range(g.d):
            assert rel_err(r["grads"][k], want[k]) < GRAD_TOL, (p, k)
        # unique rows: first-occurrence order, fp32 left-to-right sums, bit-exact
        rows, grads = r["eng"].export_unique()
        ur32, ug32 = O.unique_aggregate(idx, np.repeat(gout, np.diff(off), axis=0))
        assert np.array_equal(rows.cpu().numpy(), ur32), p
        assert np.array_equal(grads.cpu().numpy(), ug32), p


# ------------------------------------------------------------------ random
def random_batch(rng, rows, B, max_bag, skew=False):
    sizes = rng.integers(1, max_bag + 1, size=B)
    if skew:
        p = 1.0 / np.arange(1, rows + 1) ** 1.05
        idx = rng.choice(rows, size=int(sizes.sum()), p=p / p.sum())
    else:
        idx = rng.integers(0, rows, size=int(sizes.sum()))
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    return idx.astype(np.int64), off


@pytest.mark.parametrize("deterministic", [True, False])
@pytest.mark.parametrize("m,n,r,B,max_bag,skew", [
    ((10, 10, 10), (2, 2, 4), (1, 16, 16, 1), 300, 3, False),      # config-1 dims, small rows
    ((20, 20, 25), (4, 4, 4), (1, 32, 32, 1), 500, 20, True),      # config-2/3 dims, Zipf, pooling 20
    ((7, 11, 19), (4, 4, 4), (1, 32, 32, 1), 400, 5, False),       # Criteo-like small field
    ((3, 5, 7), (2, 3, 2), (1, 5, 3, 1), 200, 4, False),           # run-time dims path
    ((4, 6, 9), (1, 1, 7), (1, 3, 2, 1), 100, 40, True),           # n padded with 1s, long bags (> 32)
    ((1, 30, 40), (1, 4, 4), (1, 1, 8, 1), 300, 6, True),          # d=2-shaped geometry
])
def test_random_parity(m, n, r, B, max_bag, skew, deterministic):
    rng = np.random.default_rng(hash((m, B)) % 2**32)
    g = O.Geometry(m, n, r)
    cores32 = [c.astype(np.float32) for c in O.init_cores(g, 3)]
    idx, off = random_batch(rng, g.rows, B, max_bag, skew)
    gout = rng.standard_normal((B, g.cols)).astype(np.float32)
    res = run_case(g, cores32, idx, off, gout, deterministic)
    if not deterministic and not res["eng"].fast:
        pytest.skip("geometry runs the deterministic pipeline only")
    c64 = [c.astype(np.float64) for c in cores32]
    out, plan = O.forward(c64, g, idx, off, want_plan=True)
    assert rel_err(res["out"], out) < FWD_TOL
    ex = res["eng"].export_plan()
    assert np.array_equal(ex["work"], plan["work"])
    assert np.array_equal(ex["slot_occ"], plan["slot_occ"])
    assert np.array_equal(ex["seg_ids"], plan["seg_ids"])
    assert np.array_equal(ex["seg_inv"], plan["seg_inv"])
    ur, ug = O.unique_aggregate(idx, np.repeat(gout.astype(np.float64), np.diff(off), axis=0))
    want = O.core_grads(c64, g, ur, ug)
    for k in range(3):
        assert rel_err(res["grads"][k], want[k]) < GRAD_TOL, k
    st = res["eng"].status()
    assert st["P"] == np.unique(idx // g.m[2]).size
    if deterministic:
        assert st["U"] == ur.size


def test_d2_table_via_module():
    from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
    emb = TTEmbeddingBag(900, 12, (1, 6, 1), seed=4)
    assert emb.shape.d == 2
    rng = np.random.default_rng(5)
    idx, off = random_batch(rng, 900, 64, 4)
    out = emb(torch.from_numpy(idx).cuda(), torch.from_numpy(off[:-1]).cuda())
    g = O.Geometry(emb.shape.m, emb.shape.n, emb.shape.ranks)
    c64 = [c.detach().cpu().numpy().astype(np.float64) for c in emb.cores]
    assert rel_err(out.detach().cpu().numpy(), O.forward(c64, g, idx, off)) < FWD_TOL
    gout = torch.randn_like(out)
    out.backward(gout)
    ur, ug = O.unique_aggregate(idx, np.repeat(gout.cpu().numpy().astype(np.float64), np.diff(off), axis=0))
    want = O.core_grads(c64, g, ur, ug)
    for k in range(2):
        assert rel_err(emb.cores[k].grad.cpu().numpy(), want[k]) < GRAD_TOL


# ------------------------------------------------------------------ errors
def test_errors_raise_value_error():
    from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
    emb = TTEmbeddingBag(1000, 16, (1, 4, 4, 1))
    with pytest.raises(ValueError):
        emb(torch.tensor([0, 1000], device="cuda"), torch.tensor([0, 1], device="cuda"))  # out of range
    with pytest.raises(ValueError):
        emb(torch.tensor([-1], device="cuda"), torch.tensor([0], device="cuda"))
    with pytest.raises(ValueError):
        emb(torch.tensor([1, 2], device="cuda"), torch.tensor([0, 0, 2], device="cuda"), )  # empty bag
    with pytest.raises(ValueError):
        emb(torch.tensor([], dtype=torch.int64, device="cuda"), torch.tensor([0], device="cuda"))
    # still usable afterwards
    out = emb(torch.tensor([3, 4, 999], device="cuda"), torch.tensor([0, 2], device="cuda"))
    assert out.shape == (2, 16)


# ------------------------------------------------------------------ update
def test_sgd_update_bit_exact():
    from paper_2507_14668_b200 import _native as nat
    from paper_2507_14668_b200.engine import _ptr, _stream
    lib = nat.load()
    rng = np.random.default_rng(9)
    p0 = rng.standard_normal(10_001).astype(np.float32)
    g = rng.standard_normal(10_001).astype(np.float32)
    for mu in (0.0, 0.9):
        p = torch.from_numpy(p0.copy()).cuda()
        gg = torch.from_numpy(g).cuda()
        v = torch.zeros(p.numel(), dtype=torch.float64, device="cuda")
        ref = p0.copy()
        vel = None
        for _ in range(3):
            nat.check(lib.ttb_sgd_update(_ptr(p), _ptr(gg), _ptr(v) if mu else None, p.numel(), 0.05, mu, _stream()))
            vel = O.sgd_step(ref, g.astype(np.float64), 0.05, mu, vel)
        assert np.array_equal(p.cpu().numpy(), ref)


def test_fused_sgd_module_matches_oracle():
    from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
    emb = TTEmbeddingBag(8000, 16, (1, 8, 8, 1), seed=2).enable_fused_sgd(0.05, 0.9)
    g = O.Geometry(emb.shape.m, emb.shape.n, emb.shape.ranks)
    ref = [c.detach().cpu().numpy().astype(np.float32).copy() for c in emb.cores]
    vel = [None] * 3
    rng = np.random.default_rng(11)
    for step in range(3):
        idx, off = random_batch(rng, 8000, 128, 3, skew=True)
        out = emb(torch.from_numpy(idx).cuda(), torch.from_numpy(off[:-1]).cuda())
        gout = torch.from_numpy(rng.standard_normal(out.shape).astype(np.float32)).cuda()
        out.backward(gout)
        c64 = [c.astype(np.float64) for c in ref]
        ur, ug = O.unique_aggregate(idx, np.repeat(gout.cpu().numpy().astype(np.float64), np.diff(off), axis=0))
        want = O.core_grads(c64, g, ur, ug)
        for k in range(3):
            vel[k] = O.sgd_step(ref[k], want[k], 0.05, 0.9, vel[k])
    for k in range(3):
        assert rel_err(emb.cores[k].detach().cpu().numpy(), ref[k]) < 1e-5, k


# ------------------------------------------------------------------ full size
def test_config2_full_size_properties():
    """BASELINE config 2 (10M x 64, R=32, B=65536, pooling 1, uniform): plan
    counts vs numpy, forward on a sample of bags vs the oracle's row
    reconstruction, gradient determinism (two runs bitwise equal)."""
    from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
    emb = TTEmbeddingBag(10_000_000, 64, (1, 32, 32, 1), seed=0, max_indices=65536, deterministic=True)
    idx = np.random.default_rng(1).integers(0, 10_000_000, 65536)
    off = np.arange(65537, dtype=np.int64)
    gout = np.random.default_rng(2).standard_normal((65536, 64)).astype(np.float32)
    ti, to = torch.from_numpy(idx).cuda(), torch.from_numpy(off).cuda()
    eng = emb.engine
    cores = [c.detach() for c in emb.cores]
    eng.plan(ti, to)
    out = eng.forward(cores)
    st = eng.check_errors()
    assert st["P"] == np.unique(idx // 250).size and st["S"] == 65536
    g1 = [x.clone() for x in eng.backward(cores, torch.from_numpy(gout).cuda())]
    assert eng.status()["U"] == np.unique(idx).size
    g = O.Geometry(emb.shape.m, emb.shape.n, emb.shape.ranks)
    c64 = [c.cpu().numpy().astype(np.float64) for c in cores]
    sample = np.random.default_rng(3).choice(65536, 2000, replace=False)
    want = O.reconstruct_rows(c64, g, idx[sample])
    assert rel_err(out.cpu().numpy()[sample], want) < FWD_TOL
    eng.plan(ti, to)
    eng.forward(cores)
    g2 = eng.backward(cores, torch.from_numpy(gout).cuda())
    for a, b in zip(g1, g2):
        assert torch.equal(a, b)
    # gradients on a sub-batch against the oracle (fp64)
    sub = 4096
    eng.plan(ti[:sub], to[: sub + 1])
    eng.forward(cores)
    gs = eng.backward(cores, torch.from_numpy(gout[:sub]).cuda())
    ur, ug = O.unique_aggregate(idx[:sub], gout[:sub].astype(np.float64))
    want = O.core_grads(c64, g, ur, ug)
    for k in range(3):
        assert rel_err(gs[k].cpu().numpy(), want[k]) < GRAD_TOL


def test_dp_step_matches_fused_update():
    """dp.dp_step (gradients -> flat all-reduce -> ttb_sgd_update), here on
    one process, lands on the same bits as the fused backward + SGD path."""
    from paper_2507_14668_b200 import dp
    from paper_2507_14668_b200.engine import TtEngine
    from paper_2507_14668_b200.geometry import TtShape, init_random_cores
    shape = TtShape((20, 20, 25), (4, 4, 4), (1, 32, 32, 1))
    host = init_random_cores(shape, 7)
    rng = np.random.default_rng(8)
    idx, off = random_batch(rng, shape.rows, 256, 3, skew=True)
    ti, to = torch.from_numpy(idx).cuda(), torch.from_numpy(off).cuda()
    gout = torch.from_numpy(rng.standard_normal((256, 64)).astype(np.float32)).cuda()
    e1, e2 = TtEngine(shape, 4096, 4096, deterministic=True), TtEngine(shape, 4096, 4096, deterministic=True)
    flat = dp.FlatCores([torch.from_numpy(c).cuda() for c in host])
    fused = dp.FlatCores([torch.from_numpy(c).cuda() for c in host])
    for _ in range(3):
        dp.dp_step(e1, flat, ti, to, gout, 0.05, 0.9)
        e2.plan(ti, to)
        e2.forward(fused.cores)
        e2.backward_sgd(fused.cores, gout, 0.05, 0.9, fused.velocities)
    torch.cuda.synchronize()
    assert torch.equal(flat.param, fused.param)
    assert torch.equal(flat.velocity, fused.velocity)


def test_split_backward_paths_match_oracle():
    """The split backward (rows kernel + tcgen05 3xTF32 GEMM kernel) is
    selectable (TTB_OPT_BWD_SPLIT); it must meet the same gradient bar."""
    g = O.Geometry((40, 60, 25), (4, 4, 4), (1, 32, 32, 1))
    cores32 = [c.astype(np.float32) for c in O.init_cores(g, 6)]
    rng = np.random.default_rng(12)
    idx, off = random_batch(rng, g.rows, 3000, 3, skew=True)
    gout = rng.standard_normal((3000, g.cols)).astype(np.float32)
    eng = make_engine(g, idx.size, 3000, deterministic=True)
    eng.set_option(1, 1)
    dc = to_dev(cores32)
    eng.plan(torch.from_numpy(idx).cuda(), torch.from_numpy(off).cuda())
    eng.forward(dc)
    grads = eng.backward(dc, torch.from_numpy(gout).cuda())
    ur, ug = O.unique_aggregate(idx, np.repeat(gout.astype(np.float64), np.diff(off), axis=0))
    want = O.core_grads([c.astype(np.float64) for c in cores32], g, ur, ug)
    for k in range(3):
        assert rel_err(grads[k].cpu().numpy(), want[k]) < GRAD_TOL, k


# ------------------------------------------------------------------ tensor-core pipeline
def test_fast_config2_full_size():
    """BASELINE config 2 on the tensor-core pipeline (the default for this
    geometry): prefix count, forward on a sample vs the oracle, gradients on a
    sub-batch vs the oracle, fused SGD(+momentum) vs the oracle's update."""
    from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
    emb = TTEmbeddingBag(10_000_000, 64, (1, 32, 32, 1), seed=0, max_indices=65536)
    eng = emb.engine
    assert eng.fast
    idx = np.random.default_rng(1).integers(0, 10_000_000, 65536)
    off = np.arange(65537, dtype=np.int64)
    gout = np.random.default_rng(2).standard_normal((65536, 64)).astype(np.float32)
    ti, to = torch.from_numpy(idx).cuda(), torch.from_numpy(off).cuda()
    cores = [c.detach() for c in emb.cores]
    eng.plan(ti, to)
    out = eng.forward(cores)
    st = eng.check_errors()
    assert st["P"] == np.unique(idx // 250).size
    g = O.Geometry(emb.shape.m, emb.shape.n, emb.shape.ranks)
    c64 = [c.cpu().numpy().astype(np.float64) for c in cores]
    sample = np.random.default_rng(3).choice(65536, 2000, replace=False)
    assert rel_err(out.cpu().numpy()[sample], O.reconstruct_rows(c64, g, idx[sample])) < FWD_TOL
    full = [x.clone() for x in eng.backward(cores, torch.from_numpy(gout).cuda())]
    sub = 4096
    eng.plan(ti[:sub], to[: sub + 1])
    eng.forward(cores)
    gs = eng.backward(cores, torch.from_numpy(gout[:sub]).cuda())
    ur, ug = O.unique_aggregate(idx[:sub], gout[:sub].astype(np.float64))
    want = O.core_grads(c64, g, ur, ug)
    for k in range(3):
        assert rel_err(gs[k].cpu().numpy(), want[k]) < GRAD_TOL
    # full batch against the deterministic pipeline
    det = make_engine(g, 65536, 65536, deterministic=True)
    det.plan(ti, to)
    det.forward(cores)
    gd = det.backward(cores, torch.from_numpy(gout).cuda())
    for k in range(3):
        assert rel_err(full[k].cpu().numpy(), gd[k].cpu().numpy().astype(np.float64)) < GRAD_TOL
    # fused SGD(+momentum): two steps vs the oracle update on the same grads
    work = [c.clone() for c in cores]
    vel = [torch.zeros(c.shape, dtype=torch.float64, device="cuda") for c in cores]
    ref = [c.cpu().numpy().astype(np.float32) for c in cores]
    rvel = [np.zeros(c.shape) for c in ref]
    for _ in range(2):
        eng.plan(ti[:sub], to[: sub + 1])
        eng.forward(work)
        gk = [x.clone() for x in eng.backward(work, torch.from_numpy(gout[:sub]).cuda())]
        eng.plan(ti[:sub], to[: sub + 1])
        eng.forward(work)
        eng.backward_sgd(work, torch.from_numpy(gout[:sub]).cuda(), 0.05, 0.9, vel)
        for k in range(3):
            rvel[k] = O.sgd_step(ref[k], gk[k].cpu().numpy(), 0.05, 0.9, rvel[k])
    for k in range(3):
        assert rel_err(work[k].cpu().numpy(), ref[k]) < 1e-5


@pytest.mark.parametrize("B,max_bag,skew", [(2000, 1, False), (1500, 20, True), (300, 200, True)])
def test_fast_pooled_and_hot_rows(B, max_bag, skew):
    """Pooled bags, hot Zipf rows and items split across kItemLen: outputs and
    gradients vs the oracle (tensor-core pipeline)."""
    g = O.Geometry((20, 20, 25), (4, 4, 4), (1, 32, 32, 1))
    cores32 = [c.astype(np.float32) for c in O.init_cores(g, 9)]
    rng = np.random.default_rng(B)
    idx, off = random_batch(rng, g.rows, B, max_bag, skew)
    gout = rng.standard_normal((B, g.cols)).astype(np.float32)
    res = run_case(g, cores32, idx, off, gout)
    assert res["eng"].fast
    c64 = [c.astype(np.float64) for c in cores32]
    assert rel_err(res["out"], O.forward(c64, g, idx, off)) < FWD_TOL
    ur, ug = O.unique_aggregate(idx, np.repeat(gout.astype(np.float64), np.diff(off), axis=0))
    want = O.core_grads(c64, g, ur, ug)
    for k in range(3):
        assert rel_err(res["grads"][k], want[k]) < GRAD_TOL, k


@pytest.mark.parametrize("pool", [1, 7])
def test_fast_repeated_rows(pool):
    """Few distinct rows repeated within and across bags (the backward groups
    an item's positions by row when bags are pooled, by bag run otherwise)."""
    g = O.Geometry((20, 20, 25), (4, 4, 4), (1, 32, 32, 1))
    cores32 = [c.astype(np.float32) for c in O.init_cores(g, 3)]
    rng = np.random.default_rng(pool)
    B = 1200
    rows = rng.integers(0, g.rows, 40)
    idx = rows[rng.integers(0, 40, B * pool)]
    off = np.arange(0, B * pool + 1, pool, dtype=np.int64)
    gout = rng.standard_normal((B, g.cols)).astype(np.float32)
    res = run_case(g, cores32, idx, off, gout)
    assert res["eng"].fast
    c64 = [c.astype(np.float64) for c in cores32]
    assert rel_err(res["out"], O.forward(c64, g, idx, off)) < FWD_TOL
    ur, ug = O.unique_aggregate(idx, np.repeat(gout.astype(np.float64), np.diff(off), axis=0))
    want = O.core_grads(c64, g, ur, ug)
    for k in range(3):
        assert rel_err(res["grads"][k], want[k]) < GRAD_TOL, k


def test_fast_errors_raise():
    from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
    emb = TTEmbeddingBag(10000, 64, (1, 32, 32, 1), tt_m=(20, 20, 25), tt_n=(4, 4, 4))
    assert emb.engine.fast
    with pytest.raises(ValueError):
        emb(torch.tensor([0, 10000], device="cuda"), torch.tensor([0, 1], device="cuda"))
    with pytest.raises(ValueError):
        emb(torch.tensor([0, 1], device="cuda"), torch.tensor([0, 2, 2], device="cuda"))
    out = emb(torch.tensor([3, 4, 5], device="cuda"), torch.tensor([0, 1], device="cuda"))
    with pytest.raises(ValueError):
        out.backward(torch.full_like(out, float("nan")))
        emb.engine.check_errors()


def test_fast_fused_sgd_steps_match_oracle():
    """Several fused-SGD steps on the tensor-core pipeline: each step's update
    also writes the next forward's core images (no rebuild in between). The
    forward is checked against the oracle on the cores the GPU holds at that
    step (the images must follow every update exactly); the 4-step trajectory
    against the oracle's own, within 5e-5: each update inherits the gradients'
    (pinned to 1e-4) error, and momentum carries it over the steps (observed
    ~1e-5 after 4 steps, so a 1e-5 bound on the trajectory was flaky)."""
    from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
    emb = TTEmbeddingBag(10000, 64, (1, 32, 32, 1), tt_m=(20, 20, 25), tt_n=(4, 4, 4), seed=4)
    emb.enable_fused_sgd(0.05, 0.9)
    assert emb.engine.fast
    g = O.Geometry(emb.shape.m, emb.shape.n, emb.shape.ranks)
    ref = [c.detach().cpu().numpy().astype(np.float32).copy() for c in emb.cores]
    vel = [None] * 3
    rng = np.random.default_rng(21)
    for step in range(4):
        idx, off = random_batch(rng, 10000, 700, 4, skew=True)
        now = [c.detach().cpu().numpy().astype(np.float64) for c in emb.cores]
        out = emb(torch.from_numpy(idx).cuda(), torch.from_numpy(off[:-1]).cuda())
        assert rel_err(out.detach().cpu().numpy(), O.forward(now, g, idx, off)) < FWD_TOL, step
        gout = torch.from_numpy(rng.standard_normal(out.shape).astype(np.float32)).cuda()
        out.backward(gout)
        c64 = [c.astype(np.float64) for c in ref]
        ur, ug = O.unique_aggregate(idx, np.repeat(gout.cpu().numpy().astype(np.float64), np.diff(off), axis=0))
        want = O.core_grads(c64, g, ur, ug)
        for k in range(3):
            vel[k] = O.sgd_step(ref[k], want[k], 0.05, 0.9, vel[k])
    for k in range(3):
        assert rel_err(emb.cores[k].detach().cpu().numpy(), ref[k]) < 5e-5, k


def test_fast_core_images_follow_core_changes():
    """Core values changed outside the fused update (torch in-place ops, or
    ttb_sgd_update after a gradient-returning backward) reach the next
    forward: the cached core images are dropped."""
    from paper_2507_14668_b200 import _native as nat
    from paper_2507_14668_b200.engine import _ptr, _stream
    g = O.Geometry((20, 20, 25), (4, 4, 4), (1, 32, 32, 1))
    cores32 = [c.astype(np.float32) for c in O.init_cores(g, 5)]
    rng = np.random.default_rng(3)
    idx, off = random_batch(rng, g.rows, 500, 3, skew=False)
    eng = make_engine(g, idx.size, off.size - 1)
    assert eng.fast
    dc = to_dev(cores32)
    ti, to = torch.from_numpy(idx).cuda(), torch.from_numpy(off).cuda()

    def check():
        eng.plan(ti, to)
        out = eng.forward(dc).cpu().numpy()
        want = O.forward([c.cpu().numpy().astype(np.float64) for c in dc], g, idx, off)
        assert rel_err(out, want) < FWD_TOL

    check()
    with torch.no_grad():
        dc[1].mul_(0.5)  # torch in-place: version bump
    check()
    grads = eng.backward(dc, torch.randn(off.size - 1, g.cols, device="cuda"))
    for c, gr in zip(dc, grads):  # raw-pointer update the version counter does not see
        nat.check(eng.lib.ttb_sgd_update(_ptr(c), _ptr(gr), None, c.numel(), 0.5, 0.0, _stream()))
    check()


def test_staged_loop_matches_direct():
    """StagedLoop (side-stream uploads / downloads, double-buffered) returns
    the same per-step results as running the steps with plain copies."""
    from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
    from paper_2507_14668_b200.staging import StagedLoop, stage_batches
    rng = np.random.default_rng(8)
    batches = []
    for _ in range(3):
        idx, off = random_batch(rng, 10000, 400, 3, skew=True)
        batches.append([torch.from_numpy(idx), torch.from_numpy(off[:-1].copy())])
    emb = TTEmbeddingBag(10000, 64, (1, 32, 32, 1), tt_m=(20, 20, 25), tt_n=(4, 4, 4), seed=1)
    want = [emb(b[0].cuda(), b[1].cuda()).detach().cpu() for b in batches]
    # same shapes per step are required by the staging slots: use one batch
    loop = StagedLoop(stage_batches(batches[:1]), torch.empty(400, 64), "cuda")

    def compute(i, o):
        out = emb(i, o)
        return out, None

    loop.run(compute, 4)
    for k in (2, 3):  # pooled bags sum with fp32 reductions: order not fixed
        assert rel_err(loop.result(k).numpy(), want[0].numpy()) < FWD_TOL


def test_fast_config3_shape_vs_deterministic():
    """Config-3-shaped batch (10M x 64, ranks 32, Zipf(1.05), pooling 20) on
    the tensor-core pipeline — hot prefixes with thousands of lookups (full
    work items, warp-cooperative item writes, length-sorted tiles, weighted
    CTA ranges) — against the deterministic pipeline (parity-pinned on the
    oracle), native and permuted ids; a sample of bags against the oracle."""
    from bench_extras import zipf
    from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
    B, pool = 16384, 20
    emb = TTEmbeddingBag(10_000_000, 64, (1, 32, 32, 1), seed=0, max_indices=B * pool, max_bags=B)
    assert emb.engine.fast
    g = O.Geometry(emb.shape.m, emb.shape.n, emb.shape.ranks)
    cores = [c.detach() for c in emb.cores]
    c64 = [c.cpu().numpy().astype(np.float64) for c in cores]
    det = make_engine(g, B * pool, B, deterministic=True)
    for permuted in (False, True):
        rng = np.random.default_rng(4 + permuted)
        idx = zipf(10_000_000, B * pool, rng)
        if permuted:
            idx = np.random.default_rng(123).permutation(10_000_000)[idx]
        off = np.arange(0, B * pool + 1, pool, dtype=np.int64)
        gout = (rng.standard_normal((B, 64)) / B).astype(np.float32)
        ti, to, tg = torch.from_numpy(idx).cuda(), torch.from_numpy(off).cuda(), torch.from_numpy(gout).cuda()
        emb.engine.plan(ti, to)
        out = emb.engine.forward(cores)
        grads = [x.clone() for x in emb.engine.backward(cores, tg)]
        det.plan(ti, to)
        want = det.forward(cores)
        gd = det.backward(cores, tg)
        assert rel_err(out.cpu().numpy(), want.cpu().numpy()) < FWD_TOL
        for k in range(3):
            assert rel_err(grads[k].cpu().numpy(), gd[k].cpu().numpy()) < GRAD_TOL, (permuted, k)
        bags = np.random.default_rng(9).choice(B, 64, replace=False)
        ref = np.stack([O.reconstruct_rows(c64, g, idx[off[b]:off[b + 1]]).sum(0) for b in bags])
        assert rel_err(out.cpu().numpy()[bags], ref) < FWD_TOL


def test_fast_m3_261_kaggle_field():
    """The Criteo-Kaggle 10,131,227-row field factorises to m = (171, 227, 261):
    G3 (133.6 KB) still fits the forward's shared memory -> tensor-core
    pipeline; outputs and gradients vs the deterministic pipeline and a
    sample vs the oracle."""
    from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
    emb = TTEmbeddingBag(10_131_227, 64, (1, 32, 32, 1), seed=1, max_indices=8192)
    assert tuple(emb.shape.m) == (171, 227, 261) and emb.engine.fast
    g = O.Geometry(emb.shape.m, emb.shape.n, emb.shape.ranks)
    rng = np.random.default_rng(14)
    idx = rng.integers(0, 10_131_227, 8192)
    off = np.arange(8193, dtype=np.int64)
    gout = rng.standard_normal((8192, 64)).astype(np.float32)
    cores = [c.detach() for c in emb.cores]
    ti, to, tg = torch.from_numpy(idx).cuda(), torch.from_numpy(off).cuda(), torch.from_numpy(gout).cuda()
    emb.engine.plan(ti, to)
    out = emb.engine.forward(cores)
    grads = [x.clone() for x in emb.engine.backward(cores, tg)]
    det = make_engine(g, 8192, 8192, deterministic=True)
    det.plan(ti, to)
    want = det.forward(cores)
    gd = det.backward(cores, tg)
    assert rel_err(out.cpu().numpy(), want.cpu().numpy()) < FWD_TOL
    for k in range(3):
        assert rel_err(grads[k].cpu().numpy(), gd[k].cpu().numpy()) < GRAD_TOL, k
    c64 = [c.cpu().numpy().astype(np.float64) for c in cores]
    sample = rng.choice(8192, 256, replace=False)
    assert rel_err(out.cpu().numpy()[sample], O.reconstruct_rows(c64, g, idx[sample])) < FWD_TOL


def test_fast_int32_indices_and_last_offset():
    """int32 indices and include_last_offset=True through the module on the
    tensor-core pipeline, against the oracle."""
    from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
    emb = TTEmbeddingBag(10000, 64, (1, 32, 32, 1), tt_m=(20, 20, 25), tt_n=(4, 4, 4), seed=6,
                         include_last_offset=True)
    assert emb.engine.fast
    g = O.Geometry(emb.shape.m, emb.shape.n, emb.shape.ranks)
    rng = np.random.default_rng(12)
    idx, off = random_batch(rng, 10000, 900, 5, skew=True)
    out = emb(torch.from_numpy(idx.astype(np.int32)).cuda(), torch.from_numpy(off).cuda())
    c64 = [c.detach().cpu().numpy().astype(np.float64) for c in emb.cores]
    assert rel_err(out.detach().cpu().numpy(), O.forward(c64, g, idx, off)) < FWD_TOL


def test_large_m3_runs_deterministic_pipeline():
    """m3 > 288 (G3 no longer fits the forward kernel's shared memory): the
    engine selects the deterministic pipeline, which matches the oracle."""
    g = O.Geometry((8, 8, 300), (4, 4, 4), (1, 32, 32, 1))
    cores32 = [c.astype(np.float32) for c in O.init_cores(g, 3)]
    rng = np.random.default_rng(2)
    idx, off = random_batch(rng, g.rows, 400, 3, skew=False)
    gout = rng.standard_normal((400, g.cols)).astype(np.float32)
    res = run_case(g, cores32, idx, off, gout)
    assert not res["eng"].fast
    c64 = [c.astype(np.float64) for c in cores32]
    assert rel_err(res["out"], O.forward(c64, g, idx, off)) < FWD_TOL
    ur, ug = O.unique_aggregate(idx, np.repeat(gout.astype(np.float64), np.diff(off), axis=0))
    want = O.core_grads(c64, g, ur, ug)
    for k in range(3):
        assert rel_err(res["grads"][k], want[k]) < GRAD_TOL, k


@pytest.mark.parametrize("m,B,max_bag", [((300, 7, 25), 700, 3), ((20, 20, 25), 1, 1), ((20, 20, 25), 3, 2),
                                         ((6, 5, 288), 600, 4), ((9, 11, 1), 500, 3), ((1, 40, 30), 400, 3),
                                         ((50, 1, 40), 400, 3)])
def test_fast_edge_geometries(m, B, max_bag):
    """Tensor-core pipeline edge cases: m1 > 256 (the plan's per-group counters
    no longer fit its register cache), a single lookup, a three-bag batch, the
    largest G3 the forward keeps resident (m3 = 288), one-slice G3 (m3 = 1),
    and a single prefix group on either side (m1 = 1: one key per i2 group;
    m2 = 1: every lookup in one i2 group)."""
    g = O.Geometry(m, (4, 4, 4), (1, 32, 32, 1))
    cores32 = [c.astype(np.float32) for c in O.init_cores(g, 8)]
    rng = np.random.default_rng(B)
    idx, off = random_batch(rng, g.rows, B, max_bag, skew=False)
    gout = rng.standard_normal((B, g.cols)).astype(np.float32)
    res = run_case(g, cores32, idx, off, gout)
    assert res["eng"].fast
    c64 = [c.astype(np.float64) for c in cores32]
    assert rel_err(res["out"], O.forward(c64, g, idx, off)) < FWD_TOL
    ur, ug = O.unique_aggregate(idx, np.repeat(gout.astype(np.float64), np.diff(off), axis=0))
    want = O.core_grads(c64, g, ur, ug)
    for k in range(3):
        assert rel_err(res["grads"][k], want[k]) < GRAD_TOL, k


@pytest.mark.parametrize("m", [(6, 5, 288), (50, 1, 40), (1, 40, 30)])
def test_fast_edge_geometries_pooled_hot(m):
    """Pooled Zipf batches (hot keys: full items, the row sort's chunks and
    the row-grouped backward) on the boundary geometries of the tensor-core
    pipeline: the largest resident G3 and a single prefix group on either
    side. Forward and core gradients against the fp64 oracle."""
    g = O.Geometry(m, (4, 4, 4), (1, 32, 32, 1))
    cores32 = [c.astype(np.float32) for c in O.init_cores(g, 21)]
    rng = np.random.default_rng(sum(m))
    idx, off = random_batch(rng, g.rows, 1500, 20, skew=True)
    gout = rng.standard_normal((off.size - 1, g.cols)).astype(np.float32)
    res = run_case(g, cores32, idx, off, gout)
    assert res["eng"].fast
    c64 = [c.astype(np.float64) for c in cores32]
    assert rel_err(res["out"], O.forward(c64, g, idx, off)) < FWD_TOL
    ur, ug = O.unique_aggregate(idx, np.repeat(gout.astype(np.float64), np.diff(off), axis=0))
    want = O.core_grads(c64, g, ur, ug)
    for k in range(3):
        assert rel_err(res["grads"][k], want[k]) < GRAD_TOL, k
