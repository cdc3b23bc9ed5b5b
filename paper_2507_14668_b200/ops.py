"""The reference's operator API (pkg/src/ttemb/lookup.py, backward.py) on the
GPU: same names, argument meaning, return shapes and ValueError behaviour,
backed by the CUDA library. Arrays come back as torch CUDA tensors.

    OpCounters, ReusePlan         lookup.py:27-76
    prepare_reuse_plan            lookup.py:97-124
    forward_batch                 lookup.py:236-296
    EmbGradBatch, CoreGrads,
    OptimizerState                backward.py:29-69
    unique_aggregate              backward.py:72-87
    tt_core_grads                 backward.py:101-183
    fused_update                  backward.py:186-204
    backward_batch                backward.py:207-227

The GPU always runs the reuse schedule (prefix products once per distinct
prefix); `use_reuse=False` is accepted for API compatibility and changes only
the reported counters, which then follow the direct path's accounting.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _native as nat
from .engine import TtEngine, _ptr, _stream, bags_to_tensors, require_cuda
from .geometry import TtShape


@dataclass
class OpCounters:
    slice_mults: int = 0
    row_adds: int = 0
    buffer_hits: int = 0
    buffer_misses: int = 0

    def add(self, other: "OpCounters") -> "OpCounters":
        self.slice_mults += other.slice_mults
        self.row_adds += other.row_adds
        self.buffer_hits += other.buffer_hits
        self.buffer_misses += other.buffer_misses
        return self

    def as_dict(self) -> dict:
        return dict(slice_mults=self.slice_mults, row_adds=self.row_adds, buffer_hits=self.buffer_hits,
                    buffer_misses=self.buffer_misses)


class GpuTtTable:
    """TT table resident on a CUDA device (cores fp32, reference layout)."""

    def __init__(self, shape: TtShape, cores, device=None):
        dev = require_cuda(device)
        self.shape = shape
        self.cores = [torch.as_tensor(np.asarray(c, dtype=np.float32) if not torch.is_tensor(c) else c)
                      .to(device=dev, dtype=torch.float32).contiguous() for c in cores]
        for k, c in enumerate(self.cores):
            if tuple(c.shape) != shape.core_extent(k):
                raise ValueError(f"core {k} extent {tuple(c.shape)} != {shape.core_extent(k)}")
            if not torch.isfinite(c).all():
                raise ValueError(f"core {k} contains non-finite entries")
        self._engine: Optional[TtEngine] = None

    @property
    def device(self):
        return self.cores[0].device

    def engine(self, T: int, B: int) -> TtEngine:
        if self._engine is None:
            # the operator API exposes the reuse buffer and the unique-row
            # aggregation, which only the deterministic pipeline keeps
            self._engine = TtEngine(self.shape, max(T, 1024), max(B, 1024), self.device, deterministic=True)
        self._engine.ensure_capacity(T, B)
        return self._engine

    def to_numpy(self):
        return [c.detach().cpu().numpy() for c in self.cores]


@dataclass
class ReusePlan:
    m: tuple
    work: list
    slot_of: dict
    n_indices: int

    @property
    def buf_len(self) -> int:
        return len(self.work)

    @property
    def misses(self) -> int:
        return len(self.work)

    @property
    def hits(self) -> int:
        return self.n_indices - len(self.work)


@dataclass
class ReuseBuffer:
    """Handle on the device-side reuse buffer of the table's engine."""

    plan: ReusePlan
    plan_id: int
    table: GpuTtTable

    @property
    def slots(self) -> torch.Tensor:
        return self.table._engine.export_slots()


def _flat(indices, device):
    idx = torch.as_tensor(np.asarray(indices, dtype=np.int64) if not torch.is_tensor(indices) else indices)
    idx = idx.to(device=device, dtype=torch.int64).reshape(-1)
    if idx.numel() == 0:
        raise ValueError("index bag must be a non-empty flat sequence")
    return idx


def prepare_reuse_plan(indices: Sequence[int], table: GpuTtTable, counters: Optional[OpCounters] = None) -> ReusePlan:
    if table.shape.d != 3:
        raise ValueError(f"reuse planning needs d=3, table has d={table.shape.d}")
    idx = _flat(indices, table.device)
    T = idx.numel()
    off = torch.tensor([0, T], dtype=torch.int64, device=table.device)
    eng = table.engine(T, 1)
    eng.plan(idx, off)
    eng.check_errors()
    ex = eng.export_plan()
    work = [tuple(int(v) for v in row) for row in ex["work"]]
    plan = ReusePlan(m=table.shape.m, work=work, slot_of={w[0]: w[3] for w in work}, n_indices=T)
    if counters is not None:
        counters.buffer_misses += plan.misses
        counters.buffer_hits += plan.hits
    return plan


def forward_batch(table: GpuTtTable, batch, use_reuse: bool = True, buffer: Optional[ReuseBuffer] = None):
    """Pooled embeddings (B, N) for a list of bags (or an (indices, offsets)
    pair with B+1 offsets) plus operation counters."""
    if isinstance(batch, tuple) and len(batch) == 2 and torch.is_tensor(batch[0]):
        idx, off = batch[0].to(table.device).reshape(-1), batch[1].to(table.device, torch.int64)
    else:
        if len(batch) == 0:
            raise ValueError("empty batch")
        for bag in batch:
            if len(bag) == 0:
                raise ValueError("index bag must be a non-empty flat sequence")
        idx, off = bags_to_tensors(batch, table.device)
    if buffer is not None and (not use_reuse or table.shape.d != 3):
        raise ValueError("prebuilt buffers require d=3 and use_reuse=True")
    eng = table.engine(idx.numel(), off.numel() - 1)
    eng.plan(idx, off)
    out = eng.forward(table.cores)
    st = eng.check_errors()
    T, B, P, S = st["T"], st["B"], st["P"], st["S"]
    if not use_reuse or table.shape.d != 3:
        return out, OpCounters(slice_mults=(table.shape.d - 1) * T, row_adds=T - B)
    if buffer is not None:
        if buffer.plan.n_indices != T:
            raise ValueError("prebuilt buffer does not match this batch")
        return out, OpCounters(slice_mults=S, row_adds=(T - S) + (S - B))
    return out, OpCounters(slice_mults=P + S, row_adds=(T - S) + (S - B), buffer_hits=T - P, buffer_misses=P)


def execute_prefix_products(table: GpuTtTable, plan: ReusePlan, counters: Optional[OpCounters] = None) -> ReuseBuffer:
    """Fills the device reuse buffer for the plan's indices (the engine keeps
    it for the following forward/backward)."""
    if table.shape.d != 3 or plan.m != table.shape.m:
        raise ValueError("plan was built for a different table geometry")
    if plan.buf_len == 0:
        raise ValueError("empty plan (batches are rejected upstream)")
    eng = table._engine
    if eng is None:
        raise ValueError("plan the batch with prepare_reuse_plan first")
    scratch = torch.empty((eng.B, eng.N), dtype=torch.float32, device=table.device)
    eng.forward(table.cores, out=scratch)
    if counters is not None:
        counters.slice_mults += plan.buf_len
    return ReuseBuffer(plan=plan, plan_id=eng.plan_id, table=table)


@dataclass
class EmbGradBatch:
    indices: object
    grads: object

    def __post_init__(self):
        idx = torch.as_tensor(np.asarray(self.indices, dtype=np.int64)) if not torch.is_tensor(self.indices) \
            else self.indices
        g = torch.as_tensor(np.asarray(self.grads)) if not torch.is_tensor(self.grads) else self.grads
        if idx.dim() != 1 or g.dim() != 2:
            raise ValueError("indices must be (T,), grads (T, N)")
        if idx.shape[0] != g.shape[0]:
            raise ValueError(f"{idx.shape[0]} indices vs {g.shape[0]} grads")
        if idx.shape[0] == 0:
            raise ValueError("empty gradient batch")
        self.indices, self.grads = idx, g


@dataclass
class CoreGrads:
    arrays: list


@dataclass
class OptimizerState:
    lr: float
    momentum: float = 0.0
    velocity: Optional[list] = None

    def __post_init__(self):
        if self.lr < 0:
            raise ValueError("learning rate must be non-negative")
        if not 0.0 <= self.momentum < 1.0:
            raise ValueError("momentum must lie in [0, 1)")


_agg_engines: dict = {}


def unique_aggregate(indices, grads):
    """(rows in first-occurrence order, per-row summed grads) on the GPU."""
    dev = require_cuda()
    idx = _flat(indices, dev)
    g = torch.as_tensor(np.asarray(grads) if not torch.is_tensor(grads) else grads).to(dev, torch.float32)
    if g.dim() != 2 or g.shape[0] != idx.numel():
        raise ValueError("indices and grads disagree in length")
    if (idx < 0).any():
        raise ValueError("negative row index")
    rows = int(idx.max().item()) + 1
    N = int(g.shape[1])
    key = (rows, N)
    eng = _agg_engines.get(key)
    if eng is None:
        # one-digit geometry: the row index is its own last digit
        eng = TtEngine(TtShape((1, 1, rows), (1, 1, N), (1, 1, 1, 1)), idx.numel(), idx.numel(), dev)
        _agg_engines.clear()
        _agg_engines[key] = eng
    T = idx.numel()
    eng.plan(idx, torch.arange(T + 1, dtype=torch.int64, device=dev))
    eng.aggregate(g.contiguous())
    eng.check_errors()
    return eng.export_unique()


def tt_core_grads(table: GpuTtTable, indices, grads, buffer: Optional[ReuseBuffer] = None,
                  counters: Optional[OpCounters] = None) -> CoreGrads:
    idx = _flat(indices, table.device)
    g = torch.as_tensor(np.asarray(grads) if not torch.is_tensor(grads) else grads).to(table.device, torch.float32)
    if g.shape != (idx.numel(), table.shape.cols):
        raise ValueError(f"need (U,) indices and (U, {table.shape.cols}) grads")
    if not torch.isfinite(g).all():
        raise ValueError("non-finite gradient")
    if buffer is not None and table.shape.d != 3:
        raise ValueError("reuse buffers exist only for d=3 tables")
    T = idx.numel()
    eng = table.engine(T, T)
    eng.plan(idx, torch.arange(T + 1, dtype=torch.int64, device=table.device))
    eng.forward(table.cores)
    st = eng.check_errors()
    out = eng.backward(table.cores, g)
    if counters is not None:
        d = table.shape.d
        u = eng.status()["U"]
        counters.slice_mults += {3: 7 if buffer is not None else 8, 2: 4}[d] * u
    return CoreGrads(out)


def fused_update(table: GpuTtTable, grads: CoreGrads, opt: OptimizerState) -> None:
    if len(grads.arrays) != table.shape.d:
        raise ValueError("core gradient count mismatch")
    gs = []
    for k, g in enumerate(grads.arrays):
        g = torch.as_tensor(np.asarray(g) if not torch.is_tensor(g) else g).to(table.device, torch.float32)
        if tuple(g.shape) != tuple(table.cores[k].shape):
            raise ValueError(f"core {k} gradient extent {tuple(g.shape)}")
        gs.append(g.contiguous())
    lib = nat.load()
    # every gradient is validated on the device before any core changes
    # (backward.py:190-194): one error word, checked for all cores first,
    # gates each core's update kernel
    err = torch.zeros(1, dtype=torch.int32, device=table.device)
    for g in gs:
        nat.check(lib.ttb_check_finite(_ptr(g), g.numel(), _ptr(err), _stream()), "check_finite")
    velocity = opt.velocity
    if opt.momentum > 0.0 and velocity is None:
        velocity = [torch.zeros(c.shape, dtype=torch.float64, device=table.device) for c in table.cores]
    for k, (core, g) in enumerate(zip(table.cores, gs)):
        v = velocity[k] if opt.momentum > 0.0 else None
        nat.check(lib.ttb_sgd_update_checked(_ptr(core), _ptr(g), _ptr(v), core.numel(), float(opt.lr),
                                             float(opt.momentum), _ptr(err), _stream()), "sgd_update")
    exc = nat.errbits_to_exception(int(err.item()))
    if exc is not None:
        raise exc
    if opt.momentum > 0.0:
        opt.velocity = velocity


def backward_batch(table: GpuTtTable, batch: EmbGradBatch, opt: OptimizerState, buffer: Optional[ReuseBuffer] = None,
                   aggregate: bool = True) -> OpCounters:
    """Aggregate + core gradients + fused SGD(+momentum), one device pass.
    The GPU always aggregates (aggregate=False changes only the counters)."""
    idx = batch.indices.to(table.device).reshape(-1)
    g = batch.grads.to(table.device, torch.float32)
    if g.shape[1] != table.shape.cols:
        raise ValueError(f"grads must be (T, {table.shape.cols})")
    T = idx.numel()
    eng = table.engine(T, T)
    eng.plan(idx, torch.arange(T + 1, dtype=torch.int64, device=table.device))
    eng.forward(table.cores)
    eng.check_errors()
    if opt.momentum > 0.0 and opt.velocity is None:
        opt.velocity = [torch.zeros(c.shape, dtype=torch.float64, device=table.device) for c in table.cores]
    eng.backward_sgd(table.cores, g, opt.lr, opt.momentum, opt.velocity)
    st = eng.check_errors()
    d = table.shape.d
    U = st["U"] if aggregate else T
    per = {3: 7 if buffer is not None else 8, 2: 4}[d]
    return OpCounters(slice_mults=per * U, row_adds=(T - st["U"]) if aggregate else 0)
