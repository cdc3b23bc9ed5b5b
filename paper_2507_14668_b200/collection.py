"""TTEmbeddingBagCollection: every TT field of a model in ONE table-batched
handle.

The reference steps its sparse fields one by one — FieldTable.lookup per
field in DlrmModel.forward (model.py:295-298) and FieldTable.grads per field
in loss_and_grads (model.py:334-338). Here the fields' tables share one plan,
one forward, one backward and one update launch: their cores are stored
stacked and zero-padded to the common row factors (include/ttb.h,
ttb_create_batched), so a tile of the tensor-core pipeline belongs to one
table and the kernels only offset its G1 rows, G2 slices and G3 slices.

Each table keeps the reference's own factorisation (factorize_dims) and
init_random cores, so table f's values are exactly those of a stand-alone
TTEmbeddingBag(rows_f, dim, ranks, seed=seeds[f]); table_cores(f) returns
its cores (views into the stacked parameters).
"""
from __future__ import annotations

import ctypes as C

import torch
from torch import nn

from . import _native as nat
from .embedding_bag import _TTBagFunction
from .engine import TtEngine, _ptr, _stream, require_cuda, to_offsets
from .geometry import TtShape, factorize_dims, init_random_cores


class BatchedTtEngine(TtEngine):
    """TtEngine over a table-batched handle: `shape` is the stacked geometry
    (nt M1, nt M2, nt M3), whose core extents are the stacked cores'."""

    def __init__(self, tables, bags_per_table: int, max_indices: int, device=None):
        self.tables = [TtShape(t.m, t.n, t.ranks) for t in tables]
        if not self.tables or len(self.tables) > 64:
            raise ValueError("need 1 to 64 tables")
        n, r = self.tables[0].n, self.tables[0].ranks
        if any(t.d != 3 or t.n != n or t.ranks != r for t in self.tables):
            raise ValueError("batched tables must share d = 3, n and ranks")
        if tuple(n) != (4, 4, 4) or tuple(r) != (1, 32, 32, 1):
            raise ValueError("table batching runs on the tensor-core pipeline: n = (4, 4, 4), ranks (1, 32, 32, 1)")
        self.M = tuple(max(t.m[k] for t in self.tables) for k in range(3))
        if self.M[2] > 288:
            raise ValueError("the largest m3 must be <= 288")
        F = len(self.tables)
        self.bags_per_table = int(bags_per_table)
        self._tgeoms = (nat.TtbGeom * F)()
        for f, t in enumerate(self.tables):
            for k in range(3):
                self._tgeoms[f].m[k], self._tgeoms[f].n[k] = int(t.m[k]), int(t.n[k])
            for k in range(4):
                self._tgeoms[f].r[k] = int(t.ranks[k])
        super().__init__(TtShape(tuple(F * v for v in self.M), n, r), max_indices, F * self.bags_per_table, device)

    @property
    def fast(self) -> bool:
        return True

    def _reserve(self, T: int, B: int) -> None:
        F = len(self.tables)
        T = max(T, F * self.bags_per_table)
        nbytes = C.c_size_t()
        nat.check(self.lib.ttb_batched_workspace_bytes(self._tgeoms, F, T, self.bags_per_table, C.byref(nbytes)),
                  "batched workspace size")
        ws = torch.empty(int(nbytes.value) + 256, dtype=torch.uint8, device=self.device)
        h = self.lib.ttb_create_batched(self._tgeoms, F, T, self.bags_per_table, _ptr(ws), ws.numel(), _stream())
        if not h:
            raise ValueError("ttb_create_batched rejected the tables / capacity")
        if self._handle:
            self.lib.ttb_destroy(self._handle)
        self._handle, self._ws = C.c_void_p(h), ws
        self.max_T, self.max_B = T, F * self.bags_per_table
        if getattr(self, "_allow_empty", False):
            self.set_option(nat.OPT_ALLOW_EMPTY, 1)

    def ensure_capacity(self, T: int, B: int) -> None:
        if B != len(self.tables) * self.bags_per_table:
            raise ValueError(f"a batched plan holds {len(self.tables)} x {self.bags_per_table} bags, got {B}")
        if T > self.max_T:
            self._reserve(max(T, int(self.max_T * 1.5)), B)

    def export_fast_plan(self) -> dict:  # (available; the per-table reference exports are not)
        return super().export_fast_plan()


class TTEmbeddingBagCollection(nn.Module):
    """Sum-pooled TT embedding bags for several fields in one batched handle.

    tables: [(num_embeddings, embedding_dim), ...] (one dim for all); each
    table factorised like the reference (factorize_dims) and initialised like
    init_random(seed=seeds[f]). forward(indices, offsets) takes every table's
    indices concatenated table by table and nt * bags_per_table bags (offsets
    as in nn.EmbeddingBag: (nt B,) starts or (nt B + 1,) with
    include_last_offset) and returns (nt, bags_per_table, dim)."""

    def __init__(self, tables, tt_ranks=(1, 32, 32, 1), seeds=None, bags_per_table: int = 1 << 14,
                 max_indices: int = 1 << 18, target_row_std: float = 0.1, include_last_offset: bool = False,
                 device=None, check_errors: bool = True, allow_empty_bags: bool = False):
        super().__init__()
        dev = require_cuda(device)
        tt_ranks = tuple(int(r) for r in tt_ranks)
        dims = {int(d) for _, d in tables}
        if len(dims) != 1:
            raise ValueError("all tables need the same embedding_dim")
        self.embedding_dim = dims.pop()
        self.num_embeddings = [int(r) for r, _ in tables]
        seeds = list(seeds) if seeds is not None else list(range(len(tables)))
        shapes = []
        for rows, dim in tables:
            m, n = factorize_dims(int(rows), int(dim), len(tt_ranks) - 1)
            shapes.append(TtShape(m, n, tt_ranks))
        self.shapes = shapes
        self.engine = BatchedTtEngine(shapes, bags_per_table, max_indices, dev)
        self.bags_per_table = int(bags_per_table)
        self.include_last_offset = include_last_offset
        self.check_errors = check_errors
        self.allow_empty_bags = bool(allow_empty_bags)
        if self.allow_empty_bags:
            self.engine.allow_empty(True)
        M, F = self.engine.M, len(shapes)
        stacked = [torch.zeros(self.engine.shape.core_extent(k), dtype=torch.float32) for k in range(3)]
        for f, (sh, sd) in enumerate(zip(shapes, seeds)):
            for k, c in enumerate(init_random_cores(sh, int(sd), target_row_std, dtype="float32")):
                w = sh.m[k] * sh.n[k]
                stacked[k][:, f * M[k] * sh.n[k]: f * M[k] * sh.n[k] + w, :] = torch.from_numpy(c)
        self.cores = nn.ParameterList([nn.Parameter(c.to(dev)) for c in stacked])
        self.fused_sgd = None
        self.velocity = None
        self.fused_adagrad = None
        self.state_sum = None

    # the optimizer options of TTEmbeddingBag
    from .embedding_bag import TTEmbeddingBag as _T
    enable_fused_sgd = _T.enable_fused_sgd
    disable_fused_sgd = _T.disable_fused_sgd
    enable_fused_adagrad = _T.enable_fused_adagrad
    del _T

    def set_bags_per_table(self, B: int) -> None:
        """Bags per table of the next batches (re-sizes the batched handle)."""
        if int(B) != self.bags_per_table:
            self.bags_per_table = self.engine.bags_per_table = int(B)
            self.engine._reserve(self.engine.max_T, 0)

    @property
    def num_tables(self) -> int:
        return len(self.shapes)

    def table_cores(self, f: int):
        """Table f's three cores in the reference layout (views into the
        stacked parameters)."""
        sh, M = self.shapes[f], self.engine.M
        return [c[:, f * M[k] * sh.n[k]: f * M[k] * sh.n[k] + sh.m[k] * sh.n[k], :]
                for k, c in enumerate(self.cores)]

    def forward(self, indices: torch.Tensor, offsets: torch.Tensor) -> torch.Tensor:
        off = to_offsets(indices, offsets, self.include_last_offset)
        out = _TTBagFunction.apply(self, indices.reshape(-1), off, *self.cores)
        return out.view(self.num_tables, self.bags_per_table, self.embedding_dim)

    def extra_repr(self) -> str:
        return f"{self.num_tables} tables, dim {self.embedding_dim}, rows {self.num_embeddings}, stacked M={self.engine.M}"
