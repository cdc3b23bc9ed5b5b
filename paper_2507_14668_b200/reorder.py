"""Offline index reordering on the GPU (reference pkg/src/ttemb/reorder.py).

The passes that touch every index of a trace run as CUDA kernels in libttb.so:

    count_frequencies   reorder.py:90-104   ttb_count_frequencies + ttb_rank_rows
                                            (u64 histogram, stable radix sort on
                                            ~count: count desc, row id asc)
    apply_bijection     reorder.py:286-296  ttb_apply_bijection (range-checked gather)

Host-side helpers keep the reference's names and semantics:

    hot_row_set         reorder.py:107-112
    build_bijection     reorder.py:239-283  (placement, given a community assignment)
    mean_distinct_prefixes reorder.py:299-309
    save/load_bijection reorder.py:312-334  ('old new' text format)

Building the co-occurrence graph and community detection (reorder.py:115-236,
O(n E) pure Python) stay in the reference: they run once, offline, on a sample.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Iterable, Sequence, Union

import numpy as np
import torch

from . import _native as nat
from .engine import _ptr, _stream, require_cuda

Batches = Union[torch.Tensor, Iterable[Sequence[int]]]


@dataclass
class FreqOrder:
    """Access counts plus the rank permutation (reorder.py:26-37), on the device."""

    counts: torch.Tensor        # row id -> access count (int64)
    rank_of: torch.Tensor       # row id -> frequency rank
    row_of_rank: torch.Tensor   # frequency rank -> row id

    @property
    def table_len(self) -> int:
        return int(self.counts.numel())


@dataclass
class IndexBijection:
    """A permutation of [0, table_len) and its inverse (reorder.py:70-87)."""

    forward: np.ndarray
    inverse: np.ndarray

    def __post_init__(self):
        self.forward = np.asarray(self.forward, dtype=np.int64)
        self.inverse = np.asarray(self.inverse, dtype=np.int64)
        n = self.forward.size
        if self.inverse.size != n or not np.array_equal(np.sort(self.forward), np.arange(n)):
            raise ValueError("forward map is not a permutation")
        if not (self.inverse[self.forward] == np.arange(n)).all():
            raise ValueError("inverse does not invert forward")

    @property
    def table_len(self) -> int:
        return int(self.forward.size)


def _flat_indices(batches: Batches, device) -> tuple[torch.Tensor, list[int] | None]:
    """Batches -> (flat int64 device tensor, per-batch lengths or None)."""
    if isinstance(batches, torch.Tensor):
        return batches.to(device=device, dtype=torch.int64).contiguous().reshape(-1), None
    arrs = [np.asarray(b, dtype=np.int64).reshape(-1) for b in batches]
    lens = [a.size for a in arrs]
    flat = np.concatenate(arrs) if arrs else np.zeros(0, dtype=np.int64)
    return torch.from_numpy(flat).to(device), lens


def count_frequencies(batches: Batches, table_len: int, device=None) -> FreqOrder:
    """Tally accesses per row and rank rows by (count desc, row id asc)."""
    if table_len < 1:
        raise ValueError("table_len must be positive")
    dev = require_cuda(device)
    lib = nat.load()
    flat, _ = _flat_indices(batches, dev)
    counts = torch.empty(table_len, dtype=torch.int64, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    s = _stream()
    nat.check(lib.ttb_count_frequencies(_ptr(flat), flat.numel(), table_len, _ptr(counts), _ptr(err), s),
              "count_frequencies")
    if int(err.item()):
        raise ValueError(f"batch index outside [0, {table_len})")
    if int(counts.max()) >= 2 ** 32:
        # the device ranking keys on a u32 count; beyond that fall back to a
        # device sort of the full int64 key (same order)
        key = -counts * table_len + torch.arange(table_len, device=dev)
        row_of_rank = torch.argsort(key)
    else:
        nbytes = C.c_size_t()
        nat.check(lib.ttb_rank_workspace_bytes(table_len, C.byref(nbytes)), "rank_workspace_bytes")
        ws = torch.empty(nbytes.value + 256, dtype=torch.uint8, device=dev)
        row_of_rank = torch.empty(table_len, dtype=torch.int64, device=dev)
        rank_of = torch.empty(table_len, dtype=torch.int64, device=dev)
        nat.check(lib.ttb_rank_rows(_ptr(counts), table_len, _ptr(row_of_rank), _ptr(rank_of), _ptr(ws),
                                    ws.numel(), s), "rank_rows")
        return FreqOrder(counts=counts, rank_of=rank_of, row_of_rank=row_of_rank)
    rank_of = torch.empty_like(row_of_rank)
    rank_of[row_of_rank] = torch.arange(table_len, device=dev)
    return FreqOrder(counts=counts, rank_of=rank_of, row_of_rank=row_of_rank)


def hot_row_set(freq: FreqOrder, hot_ratio: float) -> set[int]:
    """Rows whose rank falls below floor(table_len * hot_ratio) (reorder.py:107-112)."""
    if not 0.0 <= hot_ratio <= 1.0:
        raise ValueError("hot_ratio must lie in [0, 1]")
    threshold = math.floor(freq.table_len * hot_ratio)
    return set(freq.row_of_rank[:threshold].cpu().tolist())


def build_bijection(community_of: np.ndarray, hot_rows: set[int], freq: FreqOrder,
                    table_len: int) -> IndexBijection:
    """Place cold rows community by community (reorder.py:239-283).

    community_of: cold node (rank - len(hot_rows)) -> community id. Hot rows
    keep their ids; communities are ordered by descending total count (ties by
    smallest member id), members by descending count (ties by ascending id),
    and fill the free positions in ascending order.
    """
    if freq.table_len != table_len:
        raise ValueError("frequency table length mismatch")
    counts = freq.counts.cpu().numpy()
    rank_of = freq.rank_of.cpu().numpy()
    community_of = np.asarray(getattr(community_of, "community_of", community_of), dtype=np.int64)
    threshold = len(hot_rows)
    hot_mask = np.zeros(table_len, dtype=bool)
    hot_mask[list(hot_rows)] = True
    cold = np.flatnonzero(~hot_mask)
    if community_of.size != cold.size:
        raise ValueError(f"{community_of.size} assigned nodes for {cold.size} cold rows")
    comm = community_of[rank_of[cold] - threshold]
    # community keys: (-total count, smallest member)
    uniq, inv = np.unique(comm, return_inverse=True)
    total = np.zeros(uniq.size, dtype=np.int64)
    np.add.at(total, inv, counts[cold])
    first = np.full(uniq.size, table_len, dtype=np.int64)
    np.minimum.at(first, inv, cold)
    comm_order = np.lexsort((first, -total))
    comm_pos = np.empty_like(comm_order)
    comm_pos[comm_order] = np.arange(comm_order.size)
    # rows: by community position, then -count, then id
    order = np.lexsort((cold, -counts[cold], comm_pos[inv]))
    forward = np.arange(table_len, dtype=np.int64)
    forward[cold[order]] = np.flatnonzero(~hot_mask)
    inverse = np.empty(table_len, dtype=np.int64)
    inverse[forward] = np.arange(table_len)
    return IndexBijection(forward=forward, inverse=inverse)


class DeviceBijection:
    """An IndexBijection resident in HBM, for relabelling batches on the fly."""

    def __init__(self, bijection: IndexBijection, device=None):
        dev = require_cuda(device)
        self.table_len = bijection.table_len
        self.forward = torch.from_numpy(bijection.forward).to(dev)
        self.inverse = torch.from_numpy(bijection.inverse).to(dev)
        self._err = torch.zeros(1, dtype=torch.int32, device=dev)

    def relabel(self, indices: torch.Tensor, check: bool = True) -> torch.Tensor:
        """out[i] = forward[indices[i]] on the device (ttb_apply_bijection)."""
        idx = indices.to(device=self.forward.device, dtype=torch.int64).contiguous()
        out = torch.empty_like(idx)
        lib = nat.load()
        nat.check(lib.ttb_apply_bijection(_ptr(self.forward), self.table_len, _ptr(idx), _ptr(out), idx.numel(),
                                          _ptr(self._err), _stream()), "apply_bijection")
        if check and int(self._err.item()):
            raise ValueError(f"batch index outside [0, {self.table_len})")
        return out


def apply_bijection(bijection: Union[IndexBijection, DeviceBijection], batches: Batches, device=None):
    """Relabel every index, preserving batch structure and order (reorder.py:286-296).

    A list of batches comes back as a list of lists (the reference's return);
    a tensor comes back as a device tensor."""
    dbij = bijection if isinstance(bijection, DeviceBijection) else DeviceBijection(bijection, device)
    flat, lens = _flat_indices(batches, dbij.forward.device)
    out = dbij.relabel(flat)
    if lens is None:
        return out
    host = out.cpu().tolist()
    res, pos = [], 0
    for n in lens:
        res.append(host[pos:pos + n])
        pos += n
    return res


def mean_distinct_prefixes(batches: Iterable[Sequence[int]], m_last: int, device=None) -> float:
    """Mean per-batch count of distinct floor(index / m_last) (reorder.py:299-309)."""
    if m_last < 1:
        raise ValueError("m_last must be positive")
    dev = require_cuda(device)
    sizes = []
    for b in batches:
        if len(b):
            t = torch.as_tensor(np.asarray(b, dtype=np.int64), device=dev)
            sizes.append(int(torch.unique(torch.div(t, m_last, rounding_mode="floor")).numel()))
    if not sizes:
        raise ValueError("no non-empty batches")
    return float(np.mean(sizes))


def save_bijection(bijection: IndexBijection, path) -> None:
    """Text format: one 'old new' pair per line, sorted by old index."""
    with open(path, "w", encoding="ascii") as fh:
        fh.write("".join(f"{old} {new}\n" for old, new in enumerate(bijection.forward.tolist())))


def load_bijection(path) -> IndexBijection:
    pairs = []
    with open(path, "r", encoding="ascii") as fh:
        for line_no, line in enumerate(fh, start=1):
            parts = line.split()
            if not parts:
                continue
            if len(parts) != 2:
                raise ValueError(f"{path}:{line_no}: expected 'old new'")
            pairs.append((int(parts[0]), int(parts[1])))
    if [old for old, _ in pairs] != list(range(len(pairs))):
        raise ValueError(f"{path}: old indices must be 0..n-1 in order")
    forward = np.array([new for _, new in pairs], dtype=np.int64)
    if not np.array_equal(np.sort(forward), np.arange(forward.size)):
        raise ValueError("forward map is not a permutation")
    inverse = np.empty_like(forward)
    inverse[forward] = np.arange(forward.size)
    return IndexBijection(forward=forward, inverse=inverse)
