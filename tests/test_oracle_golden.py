"""Pins the CPU oracle (oracle/ttb_oracle.py) against golden vectors produced
by the unmodified reference (tests/golden/make_golden.py) and against the
known-answer vectors of the reference's own tests. CPU only."""
import numpy as np
import pytest

from oracle import ttb_oracle as O


def geom(s, p):
    return O.Geometry(tuple(int(v) for v in s[f"{p}.m"]), tuple(int(v) for v in s[f"{p}.n"]),
                      tuple(int(v) for v in s[f"{p}.r"]))


def cores(s, p, d):
    return [s[f"{p}.core{k}"] for k in range(d)]


def test_factorize_matches_reference(golden):
    s = golden("factorize")
    for d, rows, *m in s["rows"]:
        got, _ = O.factorize(int(rows), 4, int(d))
        assert got == [int(v) for v in m[:d]], (d, rows)
    for d, c, *n in s["cols"]:
        if n[0] == -1:
            with pytest.raises(ValueError):
                O.factorize(100, int(c), int(d))
        else:
            _, got = O.factorize(100, int(c), int(d))
            assert got == [int(v) for v in n[:d]]


def test_factorize_frozen_examples():
    # test_tt_core.py:94-100 and test_model.py:174-177 known answers
    assert O.factorize(1000, 64, 3) == ([10, 10, 10], [4, 4, 4])
    assert O.factorize(7, 8, 3) == ([2, 2, 2], [2, 2, 2])
    assert O.factorize(100, 16, 2) == ([10, 10], [4, 4])
    assert O.factorize(10_000_000, 64, 3) == ([200, 200, 250], [4, 4, 4])
    assert O.factorize(1_000_000, 16, 3) == ([100, 100, 100], [2, 2, 4])


def test_digits_match_reference(golden):
    s = golden("factorize")
    for row in s["digits"]:
        d = int(row[0])
        m = [int(v) for v in row[1:1 + d]]
        i = int(row[4])
        want = [int(v) for v in row[5:5 + d]]
        got = [int(x[0]) for x in O.digits_of(np.array([i]), m)]
        assert got == want
    assert [int(x[0]) for x in O.digits_of(np.array([5]), [2, 3, 2])] == [0, 2, 1]


def test_init_bit_identical(golden):
    s = golden("init")
    for j in range(4):
        rows, dim, seed, d = (int(v) for v in s[f"c{j}.args"])
        g = geom(s, f"c{j}")
        got = O.init_cores(g, seed, dtype=np.float32)
        for k in range(d):
            assert np.array_equal(got[k], s[f"c{j}.core{k}"])


def test_plan_frozen_vectors(golden):
    s = golden("forward")
    m = (2, 2, 2)
    want_work = {
        0: [(0, 0, 0, 0)],
        1: [(3, 1, 1, 0), (1, 0, 1, 1), (0, 0, 0, 2)],
    }
    for j in range(4):
        idx = s[f"frozen{j}.idx"]
        work, slot_occ = O.reuse_plan(idx, m)
        assert np.array_equal(work, s[f"frozen{j}.work"])
        hits, misses = s[f"frozen{j}.hits_misses"]
        assert work.shape[0] == misses and idx.size - work.shape[0] == hits
        if j in want_work:
            assert [tuple(r) for r in work.tolist()] == want_work[j]


def test_forward_and_plan_match_reference(golden):
    s = golden("forward")
    for c in range(int(s["ncases"])):
        p = f"case{c}"
        g = geom(s, p)
        cs = cores(s, p, g.d)
        idx, off = s[f"{p}.idx"], s[f"{p}.off"]
        out, plan = O.forward(cs, g, idx, off, want_plan=True)
        want = s[f"{p}.out"]
        tol = 1e-12 if cs[0].dtype == np.float64 else 1e-5
        scale = max(1e-3, float(np.abs(want).max()))
        assert np.abs(out - want).max() / scale < tol, p
        if g.d == 3:
            assert np.array_equal(plan["work"], s[f"{p}.work"])
            assert np.array_equal(plan["slot_occ"], s[f"{p}.slot_occ"])
            assert np.array_equal(plan["seg_ids"], s[f"{p}.seg_ids"])
            assert np.array_equal(plan["seg_inv"], s[f"{p}.seg_inv"])
            np.testing.assert_allclose(plan["slots"], s[f"{p}.slots"], rtol=1e-5 if tol > 1e-9 else 1e-12, atol=1e-7)
            cnt = O.counters_forward(plan["T"], plan["B"], plan["P"], plan["S"])
            assert [cnt[k] for k in ("slice_mults", "row_adds", "buffer_hits", "buffer_misses")] == \
                s[f"{p}.counters"].tolist()


def test_unique_aggregate_matches_reference(golden):
    s = golden("backward")
    rows, g = O.unique_aggregate([3, 1, 3, 0], np.array([[1.0, 0.0], [0.0, 1.0], [2.0, 2.0], [5.0, 5.0]]))
    assert np.array_equal(rows, s["ua_frozen.rows"]) and np.array_equal(g, s["ua_frozen.grads"])
    # exact left-to-right accumulation (test_backward.py:68-74)
    _, v = O.unique_aggregate([7, 7, 7, 7], np.array([[1e16], [1.0], [-1e16], [1.0]]))
    assert v[0, 0] == ((1e16 + 1.0) + -1e16) + 1.0
    for c in range(int(s["ncases"])):
        p = f"case{c}"
        idx, off, gout = s[f"{p}.idx"], s[f"{p}.off"], s[f"{p}.gout"]
        per = np.repeat(gout, np.diff(off), axis=0)
        r, gg = O.unique_aggregate(idx, per)
        assert np.array_equal(r, s[f"{p}.urows"])
        assert np.array_equal(gg, s[f"{p}.ugrads"])  # same order, same dtype: bit-exact


def test_core_grads_and_update_match_reference(golden):
    s = golden("backward")
    for c in range(int(s["ncases"])):
        p = f"case{c}"
        g = geom(s, p)
        cs = cores(s, p, g.d)
        borrowed = None
        if g.d == 3:  # the reference passes the forward's reuse buffer
            _, plan = O.forward(cs, g, s[f"{p}.idx"], s[f"{p}.off"], want_plan=True)
            borrowed = (plan["work"], plan["slots"])
        grads = O.core_grads(cs, g, s[f"{p}.urows"], s[f"{p}.ugrads"], borrowed=borrowed)
        for k in range(g.d):
            want = s[f"{p}.grad{k}"]
            scale = max(1e-3, float(np.abs(want).max()))
            assert np.abs(grads[k] - want).max() / scale < 1e-12, (p, k)
        for mu in (0.0, 0.9):
            cc = [x.copy() for x in cs]
            vel = [None] * g.d
            for _ in range(2):
                for k in range(g.d):
                    vel[k] = O.sgd_step(cc[k], grads[k], 0.05, mu, vel[k])
            for k in range(g.d):
                want = s[f"{p}.upd{int(mu * 10)}.core{k}"]
                if cs[0].dtype == np.float32:
                    # same fp64 grads up to 1e-12 -> same rounding except at ties
                    np.testing.assert_allclose(cc[k], want, rtol=1e-6, atol=1e-7)
                else:
                    np.testing.assert_allclose(cc[k], want, rtol=1e-12, atol=1e-13)


def test_sgd_single_rounding_exact():
    # test_backward.py:183-193: f32(f64(core) - lr * g), one rounding
    rng = np.random.default_rng(89)
    c64 = rng.standard_normal((3, 20, 4))
    c32 = c64.astype(np.float32)
    g = rng.standard_normal(c64.shape)
    O.sgd_step(c32, g, 0.01)
    assert (c32 == (c64.astype(np.float32).astype(np.float64) - 0.01 * g).astype(np.float32)).all()


def test_counter_laws():
    b = O.counters_backward(T=10, U=6, d=3, with_buffer=True)
    assert b["slice_mults"] == 42 and b["row_adds"] == 4
    assert O.counters_backward(T=10, U=6, d=3, with_buffer=False)["slice_mults"] == 48


@pytest.mark.parametrize("name,rows,ranks,bs", [("dlrm", (4000, 500, 118), (1, 4, 4, 1), 32),
                                                 ("dlrm_tc", (12000, 700), (1, 32, 32, 1), 64)])
def test_dlrm_oracle_matches_reference_run(golden, name, rows, ranks, bs):
    """oracle/dlrm_oracle.py (the CPU DLRM step bench.py times for configs 1
    and 4) reproduces the reference's train_step bit for bit: three SGD +
    momentum steps from the reference's initial parameters."""
    from oracle import dlrm_oracle as D
    z = golden(name)
    params = {k[5:]: np.array(v) for k, v in z.items() if k.startswith("init.")}
    emb = params["top.0.w"].shape[0] - len(rows) * (len(rows) + 1) // 2
    fields = []
    for f, r in enumerate(rows):
        if f"field_{f}.core0" in params:
            m, n = O.factorize(r, emb, 3)
            fields.append(O.Geometry(tuple(m), tuple(n), ranks))
        else:
            fields.append(None)
    vel = {}
    for step in range(3):
        sp = []
        for f in range(len(rows)):
            i, o = z[f"data.idx{f}"], z[f"data.off{f}"]
            a, b = o[step * bs], o[(step + 1) * bs]
            sp.append((i[a:b], o[step * bs:(step + 1) * bs + 1] - a))
        sl = slice(step * bs, (step + 1) * bs)
        loss = D.train_step(params, fields, z["data.dense"][sl], sp, z["data.labels"][sl], 0.05, 0.9, vel)
        assert loss == z["losses"][step]
        for k, p in params.items():
            assert np.array_equal(p, z[f"step{step}.{k}"]), (step, k)


def test_adagrad_oracle_matches_torch_adagrad():
    """oracle.adagrad_step restates torch.optim.Adagrad (the reference has no
    Adagrad): three steps in float64 agree with torch bit for bit, and an
    fp32 core rounds once from the fp64 update."""
    import torch
    rng = np.random.default_rng(3)
    p64 = rng.standard_normal(1000)
    p = torch.tensor(p64.copy(), dtype=torch.float64, requires_grad=True)
    opt = torch.optim.Adagrad([p], lr=0.05, eps=1e-10)
    mine, state = p64.copy(), None
    for _ in range(3):
        g = rng.standard_normal(1000)
        p.grad = torch.tensor(g)
        opt.step()
        state = O.adagrad_step(mine, g, 0.05, 1e-10, state)
        assert np.array_equal(mine, p.detach().numpy())
    c32 = p64.astype(np.float32)
    g = rng.standard_normal(1000).astype(np.float32)
    s = O.adagrad_step(c32, g, 0.05)
    g64 = g.astype(np.float64)
    want = (p64.astype(np.float32).astype(np.float64) + (-0.05 * g64) / (np.sqrt(g64 * g64) + 1e-10)).astype(np.float32)
    assert np.array_equal(c32, want) and np.array_equal(s, g64 * g64)
    with pytest.raises(ValueError):
        O.adagrad_step(c32, np.full(1000, np.nan), 0.05)
