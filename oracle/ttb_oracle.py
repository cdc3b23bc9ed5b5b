"""CPU oracle for the TT-EmbeddingBag hot path — TEST INFRASTRUCTURE ONLY.

This module restates, in numpy, the algorithm of the Rec-AD reference
artifact (pkg/src/ttemb, pure numpy) for the path the CUDA library
implements. It exists to CHECK the GPU path and to provide the CPU baseline
timing in bench.py. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import it; the product package
(paper_2507_14668_b200) never does, and fails loudly without its CUDA
library instead of falling back here.

Pinning: tests/test_oracle_golden.py checks every function below against
golden vectors produced by running the unmodified reference in the build
container (tests/golden/make_golden.py, committed with its outputs) and
against the known-answer vectors of the reference's own tests.

Each function cites the reference file:line it follows.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Geometry", "factorize", "digits_of", "init_cores", "reuse_plan", "segments",
    "forward", "forward_direct", "unique_aggregate", "core_grads", "sgd_step", "adagrad_step",
    "counters_forward", "counters_backward", "reconstruct_rows",
    "count_frequencies", "build_bijection", "apply_bijection",
]


# ------------------------------------------------------------------ geometry
@dataclass(frozen=True)
class Geometry:
    """Row factors m, column factors n, ranks r (tt_core.py:41-82)."""

    m: tuple
    n: tuple
    r: tuple

    @property
    def d(self) -> int:
        return len(self.m)

    @property
    def rows(self) -> int:
        return int(np.prod(self.m))

    @property
    def cols(self) -> int:
        return int(np.prod(self.n))

    def extent(self, k: int) -> tuple:
        return (self.r[k], self.m[k] * self.n[k], self.r[k + 1])


def _ordered_factorings(total, parts, lo, hi, floor):
    """All non-decreasing `parts`-tuples with product `total`, entries in
    [max(lo, floor), hi] — tt_core.py:143-154."""
    if parts == 1:
        if max(lo, floor) <= total <= hi:
            yield (total,)
        return
    f = max(lo, floor)
    while f <= hi and f ** parts <= total:
        if total % f == 0:
            for tail in _ordered_factorings(total // f, parts - 1, lo, hi, f):
                yield (f,) + tail
        f += 1


def _pick_balanced(cands):
    """Smallest (max - min), then lexicographic — tt_core.py:157-163."""
    cands = list(cands)
    if not cands:
        return None
    return min(cands, key=lambda t: (max(t) - min(t), t))


def factorize(rows: int, cols: int, d: int):
    """Near-balanced (m, n) factor lists — tt_core.py:166-207."""
    if d not in (2, 3):
        raise ValueError("d must be 2 or 3")
    if rows < 1 or cols < 1:
        raise ValueError("extents must be positive")
    root = rows ** (1.0 / d)
    lo = max(1, math.ceil(root / 2.0))
    hi = max(1, math.floor(root * 2.0))
    limit = math.ceil(root) ** d
    m = None
    total = rows
    while total <= limit and m is None:
        m = _pick_balanced(_ordered_factorings(total, d, lo, hi, 1))
        total += 1
    if m is None:
        raise ValueError("no row factorization")
    n = _pick_balanced(_ordered_factorings(cols, d, 2, cols, 1))
    if n is None:
        if cols >= 2 ** d:
            raise ValueError("no column factorization with factors >= 2")
        n = _pick_balanced(_ordered_factorings(cols, d, 1, cols, 1))
        if n is None:
            raise ValueError("no column factorization")
    return list(m), list(n)


def digits_of(idx, m):
    """Big-endian mixed-radix digits, vectorised — tt_core.py:210-224,
    lookup.py:214-219. Returns a list of d int64 arrays."""
    rest = np.asarray(idx, dtype=np.int64)
    out = []
    for radix in m[::-1]:
        out.append(rest % radix)
        rest = rest // radix
    return out[::-1]


def init_cores(g: Geometry, seed: int, target_row_std: float = 0.1, dtype=np.float64):
    """Scaled Gaussian cores from one PCG64 stream — tt_core.py:298-322."""
    if target_row_std <= 0:
        raise ValueError("target_row_std must be positive")
    inner = g.r[1:-1]
    rbar = float(np.mean(inner)) if len(inner) else 1.0
    sigma = target_row_std ** (1.0 / g.d) / rbar ** ((g.d - 1) / (2.0 * g.d))
    gen = np.random.default_rng(seed)
    return [(gen.standard_normal(g.extent(k)) * sigma).astype(dtype) for k in range(g.d)]


def _slice(core, nk, i):
    """Fixed-digit blocks (U, R_prev, n_k, R_next) — tt_core.py:239-248."""
    cols = np.asarray(i)[:, None] * nk + np.arange(nk)[None, :]
    return np.transpose(core[:, cols, :], (1, 0, 2, 3))


def reconstruct_rows(cores, g: Geometry, idx):
    """Dense rows by left-to-right chaining — tt_core.py:251-265."""
    idx = np.asarray(idx, dtype=np.int64)
    dg = digits_of(idx, g.m)
    acc = _slice(cores[0], g.n[0], dg[0])[:, 0]  # (T, n0, r1)
    for k in range(1, g.d):
        blk = _slice(cores[k], g.n[k], dg[k])  # (T, r, n, s)
        acc = np.einsum("tar,trns->tans", acc, blk).reshape(idx.size, -1, g.r[k + 1])
    return acc.reshape(idx.size, g.cols)


# ---------------------------------------------------------------- planning
def _validate(idx, offsets, rows):
    """Bag checks of lookup.py:88-94, 254-255 on an (indices, offsets) batch."""
    idx = np.asarray(idx, dtype=np.int64)
    offsets = np.asarray(offsets, dtype=np.int64)
    if offsets.size < 2:
        raise ValueError("empty batch")
    if offsets[0] != 0 or offsets[-1] != idx.size or (np.diff(offsets) < 0).any():
        raise ValueError("malformed offsets")
    if (np.diff(offsets) == 0).any():
        raise ValueError("index bag must be a non-empty flat sequence")
    if idx.size and ((idx < 0).any() or (idx >= rows).any()):
        raise ValueError(f"bag index outside [0, {rows})")
    return idx, offsets


def reuse_plan(idx, m):
    """First-occurrence prefix slots — lookup.py:97-124.
    Returns work (P x 4 int64: key, i1, i2, slot) and the slot of each index."""
    if len(m) != 3:
        raise ValueError("reuse planning needs d=3")
    keys = np.asarray(idx, dtype=np.int64) // m[2]
    uniq, first = np.unique(keys, return_index=True)
    order = np.argsort(first, kind="stable")
    ordered = uniq[order]  # keys in first-occurrence order
    slot_of_key = np.empty(uniq.size, dtype=np.int64)
    slot_of_key[order] = np.arange(uniq.size)
    slot_occ = slot_of_key[np.searchsorted(uniq, keys)]
    work = np.stack([ordered, ordered // m[1], ordered % m[1], np.arange(ordered.size)], axis=1)
    return work.astype(np.int64), slot_occ.astype(np.int64)


def segments(bag_ids, slot_occ, n_slots):
    """np.unique of bag * P + slot — lookup.py:280-284."""
    key = np.asarray(bag_ids, dtype=np.int64) * n_slots + np.asarray(slot_occ, dtype=np.int64)
    seg_ids, seg_inv = np.unique(key, return_inverse=True)
    return seg_ids, seg_inv.reshape(-1)


# ------------------------------------------------------------------ forward
def forward(cores, g: Geometry, idx, offsets, want_plan: bool = False):
    """Reuse forward for d=3 (lookup.py:236-296); direct chain for d=2 or as
    a fallback (lookup.py:209-233). Computes in the cores' dtype."""
    idx, offsets = _validate(idx, offsets, g.rows)
    n_bags = offsets.size - 1
    bag_ids = np.repeat(np.arange(n_bags, dtype=np.int64), np.diff(offsets))
    if g.d != 3:
        out = forward_direct(cores, g, idx, bag_ids, n_bags)
        return (out, None) if want_plan else out
    work, slot_occ = reuse_plan(idx, g.m)
    P = work.shape[0]
    n1, n2, n3 = g.n
    # prefix products (lookup.py:139-146)
    left = cores[0][0, work[:, 1][:, None] * n1 + np.arange(n1)[None, :], :]          # (P, n1, r1)
    mid = _slice(cores[1], n2, work[:, 2])                                             # (P, r1, n2, r2)
    slots = np.einsum("pxr,prys->pxys", left, mid).reshape(P, n1 * n2, g.r[2])
    slots = np.ascontiguousarray(slots)
    # per-segment G3 sums, close, pool (lookup.py:280-293)
    seg_ids, seg_inv = segments(bag_ids, slot_occ, P)
    tail = np.transpose(cores[2][:, (idx % g.m[2])[:, None] * n3 + np.arange(n3)[None, :], 0], (1, 0, 2))
    summed = np.zeros((seg_ids.size,) + tail.shape[1:], dtype=cores[2].dtype)
    np.add.at(summed, seg_inv, tail)
    closed = np.einsum("sxr,srj->sxj", slots[seg_ids % P], summed)
    out = np.zeros((n_bags, g.cols), dtype=cores[0].dtype)
    np.add.at(out, seg_ids // P, closed.reshape(seg_ids.size, g.cols))
    if not want_plan:
        return out
    plan = dict(work=work, slot_occ=slot_occ, seg_ids=seg_ids, seg_inv=seg_inv, slots=slots,
                bag_ids=bag_ids, P=P, S=int(seg_ids.size), T=int(idx.size), B=n_bags)
    return out, plan


def forward_direct(cores, g: Geometry, idx, bag_ids, n_bags):
    """No-reuse path — lookup.py:209-233."""
    rows = reconstruct_rows(cores, g, idx)
    out = np.zeros((n_bags, g.cols), dtype=cores[0].dtype)
    np.add.at(out, np.asarray(bag_ids, dtype=np.int64), rows)
    return out


# ----------------------------------------------------------------- backward
def unique_aggregate(idx, grads):
    """Rows in first-occurrence order, gradients summed left to right in the
    gradient dtype — backward.py:72-87."""
    idx = np.asarray(idx, dtype=np.int64)
    grads = np.asarray(grads)
    if idx.shape[0] != grads.shape[0]:
        raise ValueError("indices and grads disagree in length")
    uniq, first, inv = np.unique(idx, return_index=True, return_inverse=True)
    acc = np.zeros((uniq.size, grads.shape[1]), dtype=grads.dtype)
    np.add.at(acc, inv.reshape(-1), grads)
    order = np.argsort(first, kind="stable")
    return uniq[order], acc[order]


def core_grads(cores, g: Geometry, idx, grads, borrowed=None):
    """Loss gradients w.r.t. every core entry, fp64 accumulation —
    backward.py:101-183 (per-row left chain x grad slice x right chain).

    borrowed: optional (work, slots) from the forward's reuse plan; as in
    backward.py:144-150 the d=3 two-core left chain is then read from the
    reuse buffer (in the table dtype) instead of recomputed in fp64."""
    idx = np.asarray(idx, dtype=np.int64)
    G = np.asarray(grads, dtype=np.float64)
    if idx.ndim != 1 or G.shape != (idx.size, g.cols):
        raise ValueError("need (U,) indices and (U, N) grads")
    if idx.size == 0:
        raise ValueError("empty row set")
    if (idx < 0).any() or (idx >= g.rows).any():
        raise ValueError("row index outside range")
    if not np.isfinite(G).all():
        raise ValueError("non-finite gradient")
    U, d = idx.size, g.d
    dg = digits_of(idx, g.m)
    blocks = [_slice(cores[k], g.n[k], dg[k]).astype(np.float64) for k in range(d)]
    # left[k]: product of blocks < k as (U, prod n_<k, r_k); right[k]: blocks > k as (U, r_{k+1}, prod n_>k)
    left = [np.ones((U, 1, 1))]
    for k in range(d - 1):
        if k == 1 and borrowed is not None:
            work, slots = borrowed
            slot_of = {int(key): s for s, key in enumerate(work[:, 0])}
            pick = np.array([slot_of[int(p)] for p in idx // g.m[2]], dtype=np.int64)
            left.append(np.asarray(slots)[pick].astype(np.float64))
            continue
        nxt = np.einsum("uar,urns->uans", left[-1], blocks[k])
        left.append(nxt.reshape(U, -1, g.r[k + 1]))
    right = [None] * d
    right[d - 1] = np.ones((U, 1, 1))
    for k in range(d - 2, -1, -1):
        nxt = np.einsum("urns,usb->urnb", blocks[k + 1], right[k + 1])
        right[k] = nxt.reshape(U, g.r[k + 1], -1)
    out = []
    before = 1
    for k in range(d):
        nk = g.n[k]
        after = g.cols // (before * nk)
        gk = G.reshape(U, before, nk, after)
        blk = np.einsum("uar,uajb,usb->urjs", left[k], gk, right[k])  # (U, r_k, n_k, r_{k+1})
        acc = np.zeros((g.m[k] * nk, g.r[k], g.r[k + 1]))
        pos = (dg[k][:, None] * nk + np.arange(nk)[None, :]).reshape(-1)
        np.add.at(acc, pos, np.transpose(blk, (0, 2, 1, 3)).reshape(U * nk, g.r[k], g.r[k + 1]))
        out.append(np.ascontiguousarray(np.transpose(acc, (1, 0, 2))))
        before *= nk
    return out


def sgd_step(core, grad, lr, momentum=0.0, velocity=None):
    """In-place SGD(+momentum), fp64 velocity, one rounding into the core —
    backward.py:186-204 and model.py:353-364. Returns the velocity."""
    g = np.asarray(grad, dtype=np.float64)
    if not np.isfinite(g).all():
        raise ValueError("non-finite gradient")
    if momentum > 0.0:
        if velocity is None:
            velocity = np.zeros(g.shape, dtype=np.float64)
        velocity *= momentum
        velocity += g
        np.subtract(core, lr * velocity, out=core, casting="same_kind")
        return velocity
    np.subtract(core, lr * g, out=core, casting="same_kind")
    return velocity


def adagrad_step(core, grad, lr, eps=1e-10, state_sum=None):
    """In-place Adagrad, fp64 squared-gradient sums, one rounding into the
    core. NOT in the reference (it has SGD(+momentum) only);
    BASELINE north_star item (3) names Adagrad, so this restates
    torch.optim.Adagrad (lr_decay = weight_decay = 0): s = fma(g, g, s);
    p += (-lr * g) / (sqrt(s) + eps). Pinned against torch.optim.Adagrad in
    float64 (tests/test_oracle_golden.py); parity to the reference: unpinned.
    Returns the state."""
    g = np.asarray(grad, dtype=np.float64)
    if not np.isfinite(g).all():
        raise ValueError("non-finite gradient")
    if state_sum is None:
        state_sum = np.zeros(g.shape, dtype=np.float64)
    # torch's addcmul_ is one fused multiply-add (s + g*g rounded once); the
    # 64-bit-mantissa long double reproduces it (the device uses __fma_rn)
    state_sum[...] = (state_sum.astype(np.longdouble) + g.astype(np.longdouble) ** 2).astype(np.float64)
    np.add(core, (-lr * g) / (np.sqrt(state_sum) + eps), out=core, casting="same_kind")
    return state_sum


# ----------------------------------------------------------------- counters
def counters_forward(T, B, P, S):
    """Logical counters of forward_batch with planning included
    (lookup.py:121-123, 148, 294-295)."""
    return dict(slice_mults=P + S, row_adds=(T - S) + (S - B), buffer_hits=T - P, buffer_misses=P)


def counters_backward(T, U, d=3, with_buffer=True):
    """backward_batch counters (backward.py:218-222, 146-182): 7U with the
    reuse buffer, 8U without, for d=3; 4U for d=2."""
    per = {3: 7 if with_buffer else 8, 2: 4}[d]
    return dict(slice_mults=per * U, row_adds=T - U, buffer_hits=0, buffer_misses=0)


# ------------------------------------------------------------ reordering
def count_frequencies(batches, table_len):
    """(counts, row_of_rank, rank_of): bincount over all batches, rows ranked
    by count descending then id ascending (reorder.py:90-104)."""
    counts = np.zeros(table_len, dtype=np.int64)
    for b in batches:
        a = np.asarray(b, dtype=np.int64)
        if a.size == 0:
            continue
        if (a < 0).any() or (a >= table_len).any():
            raise ValueError(f"batch index outside [0, {table_len})")
        counts += np.bincount(a, minlength=table_len)
    row_of_rank = np.array(sorted(range(table_len), key=lambda r: (-int(counts[r]), r)), dtype=np.int64)
    rank_of = np.empty(table_len, dtype=np.int64)
    rank_of[row_of_rank] = np.arange(table_len)
    return counts, row_of_rank, rank_of


def build_bijection(community_of, hot_rows, counts, rank_of, table_len):
    """forward map: hot rows fixed, cold rows grouped by community, communities
    by (-total count, min member), members by (-count, id), placed on the free
    positions in ascending order (reorder.py:239-283)."""
    thr = len(hot_rows)
    groups = {}
    for row in range(table_len):
        if row not in hot_rows:
            groups.setdefault(int(community_of[int(rank_of[row]) - thr]), []).append(row)
    comms = sorted(groups.values(), key=lambda rows: (-sum(int(counts[r]) for r in rows), min(rows)))
    forward = np.full(table_len, -1, dtype=np.int64)
    for row in hot_rows:
        forward[row] = row
    free = iter(sorted(set(range(table_len)) - set(hot_rows)))
    for rows in comms:
        for row in sorted(rows, key=lambda r: (-int(counts[r]), r)):
            forward[row] = next(free)
    return forward


def apply_bijection(forward, batches):
    """Relabel every index through forward (reorder.py:286-296)."""
    out = []
    n = len(forward)
    for b in batches:
        a = np.asarray(b, dtype=np.int64)
        if a.size and ((a < 0).any() or (a >= n).any()):
            raise ValueError(f"batch index outside [0, {n})")
        out.append(np.asarray(forward)[a].tolist())
    return out
