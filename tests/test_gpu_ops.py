"""The operator-level drop-in (paper_2507_14668_b200/ops.py) against the
reference's own outputs (tests/golden/forward.npz, backward.npz, produced by
the unmodified lookup.py / backward.py).

Same names and argument meaning as the reference: forward_batch
(lookup.py:236-296), prepare_reuse_plan (lookup.py:97-124),
execute_prefix_products (lookup.py:127-149), unique_aggregate
(backward.py:72-87), tt_core_grads (backward.py:101-183), fused_update
(backward.py:186-204), backward_batch (backward.py:207-227). Integer outputs
and counters bit-exact; fp32 results within the north-star tolerances."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

FWD_TOL = 1e-5
GRAD_TOL = 1e-4


def rel_err(got, want, floor=1e-3):
    got = np.asarray(got.cpu().numpy() if torch.is_tensor(got) else got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    return float(np.abs(got - want).max() / max(floor, float(np.abs(want).max())))


def table_of(s, p):
    from paper_2507_14668_b200 import ops
    from paper_2507_14668_b200.geometry import TtShape
    m, n, r = (tuple(int(v) for v in s[f"{p}.{k}"]) for k in "mnr")
    d = len(m)
    return ops.GpuTtTable(TtShape(m, n, r), [s[f"{p}.core{k}"] for k in range(d)]), d


def bags_of(s, p):
    idx, off = s[f"{p}.idx"], s[f"{p}.off"]
    return [idx[off[b]:off[b + 1]].tolist() for b in range(off.size - 1)]


def test_forward_batch_and_counters(golden):
    from paper_2507_14668_b200 import ops
    s = golden("forward")
    for c in range(int(s["ncases"])):
        p = f"case{c}"
        table, d = table_of(s, p)
        batch = bags_of(s, p)
        out, cnt = ops.forward_batch(table, batch)
        assert rel_err(out, s[f"{p}.out"]) < FWD_TOL, p
        want = s[f"{p}.counters"]
        assert [cnt.slice_mults, cnt.row_adds, cnt.buffer_hits, cnt.buffer_misses] == want.tolist(), p
        # use_reuse=False: the reference's direct path (lookup.py:264-270) — same
        # values within tolerance and the direct path's counters
        out_d, cd = ops.forward_batch(table, batch, use_reuse=False)
        assert rel_err(out_d, s[f"{p}.out_direct"]) < FWD_TOL, p
        T, B = int(s[f"{p}.idx"].size), len(batch)
        assert (cd.slice_mults, cd.row_adds, cd.buffer_hits, cd.buffer_misses) == ((d - 1) * T, T - B, 0, 0), p


def test_prepare_plan_and_prefix_products(golden):
    from paper_2507_14668_b200 import ops
    s = golden("forward")
    n = 0
    for c in range(int(s["ncases"])):
        p = f"case{c}"
        table, d = table_of(s, p)
        if d != 3:
            with pytest.raises(ValueError):
                ops.prepare_reuse_plan(s[f"{p}.idx"], table)
            continue
        cnt = ops.OpCounters()
        plan = ops.prepare_reuse_plan(s[f"{p}.idx"], table, cnt)
        work = s[f"{p}.work"]
        assert np.array_equal(np.array(plan.work, dtype=np.int64).reshape(-1, 4), work), p
        assert plan.slot_of == {int(w[0]): int(w[3]) for w in work}
        assert (cnt.buffer_misses, cnt.buffer_hits) == (work.shape[0], s[f"{p}.idx"].size - work.shape[0])
        buf = ops.execute_prefix_products(table, plan, cnt)
        assert cnt.slice_mults == work.shape[0]
        assert rel_err(buf.slots, s[f"{p}.slots"]) < FWD_TOL, p
        # the prebuilt buffer serves forward_batch: closing-stage counters only
        out, c2 = ops.forward_batch(table, bags_of(s, p), buffer=buf)
        assert rel_err(out, s[f"{p}.out"]) < FWD_TOL
        want = s[f"{p}.counters"]
        assert c2.slice_mults == want[0] - work.shape[0] and c2.buffer_misses == 0
        n += 1
    assert n >= 10


def test_unique_aggregate(golden):
    from paper_2507_14668_b200 import ops
    b = golden("backward")
    rows, grads = ops.unique_aggregate(np.array([3, 1, 3, 0]), np.array([[1., 0.], [0., 1.], [2., 2.], [5., 5.]]))
    assert rows.cpu().numpy().tolist() == b["ua_frozen.rows"].tolist()
    assert np.array_equal(grads.cpu().numpy(), b["ua_frozen.grads"].astype(np.float32))
    for c in range(int(b["ncases"])):
        p = f"case{c}"
        idx, off = b[f"{p}.idx"], b[f"{p}.off"]
        per_occ = np.repeat(b[f"{p}.gout"], np.diff(off), axis=0).astype(np.float32)
        rows, grads = ops.unique_aggregate(idx, per_occ)
        assert np.array_equal(rows.cpu().numpy(), b[f"{p}.urows"]), p
        assert rel_err(grads, b[f"{p}.ugrads"]) < 1e-6, p
    with pytest.raises(ValueError):
        ops.unique_aggregate(np.array([1, 2]), np.ones((3, 4), np.float32))


def test_tt_core_grads(golden):
    from paper_2507_14668_b200 import ops
    b = golden("backward")
    for c in range(int(b["ncases"])):
        p = f"case{c}"
        table, d = table_of(b, p)
        cnt = ops.OpCounters()
        cg = ops.tt_core_grads(table, b[f"{p}.urows"], b[f"{p}.ugrads"].astype(np.float32), counters=cnt)
        for k in range(d):
            assert rel_err(cg.arrays[k], b[f"{p}.grad{k}"]) < GRAD_TOL, (p, k)
        # the golden run borrowed the forward's reuse buffer for d = 3 (7U mults)
        U = b[f"{p}.urows"].size
        assert cnt.slice_mults == {3: 8, 2: 4}[d] * U
        if d == 3:
            c7 = ops.OpCounters()
            plan = ops.prepare_reuse_plan(b[f"{p}.idx"], table)
            buf = ops.execute_prefix_products(table, plan)
            ops.tt_core_grads(table, b[f"{p}.urows"], b[f"{p}.ugrads"].astype(np.float32), buffer=buf, counters=c7)
            assert c7.slice_mults == int(b[f"{p}.mults"]) == 7 * U
    table, _ = table_of(b, "case1")
    bad = b["case1.ugrads"].astype(np.float32).copy()
    bad[0, 0] = np.nan
    with pytest.raises(ValueError):
        ops.tt_core_grads(table, b["case1.urows"], bad)


@pytest.mark.parametrize("mu", [0.0, 0.9])
def test_fused_update_and_backward_batch(golden, mu):
    """fused_update twice with the golden gradients (the reference's
    upd0 / upd9 snapshots), and backward_batch = aggregate + grads + update."""
    from paper_2507_14668_b200 import ops
    b = golden("backward")
    for c in range(int(b["ncases"])):
        p = f"case{c}"
        table, d = table_of(b, p)
        if any(b[f"{p}.core{k}"].dtype != np.float32 for k in range(d)):
            continue  # fp64 reference tables: the bit-exact update bar applies to fp32 cores
        opt = ops.OptimizerState(lr=0.05, momentum=mu)
        grads = ops.CoreGrads([b[f"{p}.grad{k}"].astype(np.float32) for k in range(d)])
        ops.fused_update(table, grads, opt)
        ops.fused_update(table, grads, opt)
        for k in range(d):
            got = table.cores[k].cpu().numpy()
            want = b[f"{p}.upd{int(mu * 10)}.core{k}"]
            # the golden update consumed the fp64 gradients, rounded to fp32
            # here: within an ulp of the reference's result
            assert rel_err(got, want) < 1e-6, (p, k)
        # backward_batch on a fresh table: aggregate + core grads + update
        table2, _ = table_of(b, p)
        idx, off = b[f"{p}.idx"], b[f"{p}.off"]
        per_occ = np.repeat(b[f"{p}.gout"], np.diff(off), axis=0).astype(np.float32)
        opt2 = ops.OptimizerState(lr=0.05, momentum=mu)
        cnt = ops.backward_batch(table2, ops.EmbGradBatch(idx, per_occ), opt2)
        U = b[f"{p}.urows"].size
        assert cnt.row_adds == idx.size - U
        for k in range(d):
            ref = b[f"{p}.core{k}"].astype(np.float64) - 0.05 * b[f"{p}.grad{k}"]
            assert rel_err(table2.cores[k], ref) < GRAD_TOL, (p, k)
