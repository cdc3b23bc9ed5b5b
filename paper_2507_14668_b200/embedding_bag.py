"""TTEmbeddingBag: the drop-in TT-compressed, sum-pooled EmbeddingBag.

Constructor arguments follow the reference's table seam (FieldTable(rows,
dim, ranks, ..., seed) at model.py:183-197, geometry from factorize_dims and
cores from init_random, tt_core.py:166-207 / 298-322): number of rows,
embedding dim, TT ranks, optional row/column factorisation. Cores are the
module's parameters, in the reference layout, so state_dict() round-trips
with the reference's table blobs (geometry.table_to_bytes).

forward(indices, offsets) -> (B, N) runs the CUDA plan + reuse forward;
backward either returns core gradients to autograd (default; needed for
data-parallel all-reduce or any torch optimizer) or, after
enable_fused_sgd(lr, momentum), applies the reference's SGD(+momentum) update
inside the backward kernels (backward_batch semantics, backward.py:207-227).
"""
from __future__ import annotations

import torch
from torch import nn

from .engine import TtEngine, bags_to_tensors, require_cuda, to_offsets
from .geometry import TtShape, factorize_dims, init_random_cores


class _TTBagFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, module, indices, offsets, *cores):
        eng = module.engine
        eng.plan(indices, offsets)
        out = eng.forward(cores)
        if module.check_errors:
            eng.check_errors()
        ctx.module = module
        ctx.plan_id = eng.plan_id
        ctx.save_for_backward(indices, offsets)
        return out

    @staticmethod
    def backward(ctx, grad_out):
        module = ctx.module
        eng = module.engine
        cores = list(module.cores)
        if eng.plan_id != ctx.plan_id:
            # the engine planned another batch since this forward: rebuild
            # this batch's plan and reuse buffer before differentiating
            indices, offsets = ctx.saved_tensors
            eng.plan(indices, offsets)
            eng.forward(cores)
        if module.fused_adagrad is not None:
            lr, eps = module.fused_adagrad
            with torch.no_grad():
                eng.backward_adagrad(cores, grad_out, lr, eps, module.state_sum)
            if module.check_errors:
                eng.check_errors()
            return (None, None, None, *([None] * len(cores)))
        if module.fused_sgd is not None:
            lr, mu = module.fused_sgd
            with torch.no_grad():
                eng.backward_sgd(cores, grad_out, lr, mu, module.velocity if mu > 0 else None)
            if module.check_errors:
                eng.check_errors()
            return (None, None, None, *([None] * len(cores)))
        grads = eng.backward(cores, grad_out)
        if module.check_errors:
            eng.check_errors()
        return (None, None, None, *grads)


class TTEmbeddingBag(nn.Module):
    """Sum-pooled TT embedding bag over `num_embeddings` rows of width
    `embedding_dim` with TT ranks `tt_ranks` = (1, R1, [R2,] 1)."""

    def __init__(self, num_embeddings: int, embedding_dim: int, tt_ranks, tt_m=None, tt_n=None, seed: int = 0,
                 target_row_std: float = 0.1, include_last_offset: bool = False, max_indices: int = 1 << 16,
                 max_bags: int | None = None, device=None, check_errors: bool = True, init: bool = True,
                 deterministic: bool = False, allow_empty_bags: bool = False):
        super().__init__()
        tt_ranks = tuple(int(r) for r in tt_ranks)
        d = len(tt_ranks) - 1
        if tt_m is None or tt_n is None:
            m, n = factorize_dims(num_embeddings, embedding_dim, d)
            tt_m = tt_m if tt_m is not None else m
            tt_n = tt_n if tt_n is not None else n
        self.shape = TtShape(tuple(tt_m), tuple(tt_n), tt_ranks)
        if self.shape.rows < num_embeddings:
            raise ValueError(f"factorized rows {self.shape.rows} cannot cover {num_embeddings}")
        if self.shape.cols != embedding_dim:
            raise ValueError(f"column factors give {self.shape.cols}, table needs {embedding_dim}")
        self.num_embeddings = int(num_embeddings)
        self.embedding_dim = int(embedding_dim)
        self.include_last_offset = include_last_offset
        self.check_errors = check_errors
        dev = require_cuda(device)
        if init:
            host = init_random_cores(self.shape, seed, target_row_std, dtype="float32")
            cores = [torch.from_numpy(c).to(dev) for c in host]
        else:
            cores = [torch.zeros(self.shape.core_extent(k), dtype=torch.float32, device=dev) for k in range(self.shape.d)]
        self.cores = nn.ParameterList([nn.Parameter(c) for c in cores])
        # deterministic=True: fixed summation order (bitwise reproducible
        # gradients); otherwise the tensor-core pipeline where supported
        self.engine = TtEngine(self.shape, max_indices, max_bags, dev, deterministic=deterministic)
        # allow_empty_bags: empty bags pool to zero rows as in torch.nn.EmbeddingBag
        # (the default keeps the reference's ValueError, lookup.py:90-91)
        self.allow_empty_bags = bool(allow_empty_bags)
        if self.allow_empty_bags:
            self.engine.allow_empty(True)
        self.fused_sgd = None
        self.velocity = None
        self.fused_adagrad = None
        self.state_sum = None

    # -------------------------------------------------------------- options
    def enable_fused_sgd(self, lr: float, momentum: float = 0.0) -> "TTEmbeddingBag":
        if lr < 0 or not 0.0 <= momentum < 1.0:
            raise ValueError("need lr >= 0 and 0 <= momentum < 1")
        self.fused_sgd = (float(lr), float(momentum))
        if momentum > 0 and self.velocity is None:
            self.velocity = [torch.zeros(c.shape, dtype=torch.float64, device=c.device) for c in self.cores]
        return self

    def disable_fused_sgd(self) -> "TTEmbeddingBag":
        self.fused_sgd = None
        return self

    def enable_fused_adagrad(self, lr: float, eps: float = 1e-10,
                             initial_accumulator_value: float = 0.0) -> "TTEmbeddingBag":
        """Adagrad (torch.optim.Adagrad semantics) applied inside the backward;
        state_sum holds the fp64 squared-gradient sums. Replaces a fused SGD."""
        if lr < 0 or eps < 0 or initial_accumulator_value < 0:
            raise ValueError("need lr, eps, initial_accumulator_value >= 0")
        self.fused_sgd = None
        self.fused_adagrad = (float(lr), float(eps))
        if self.state_sum is None:
            self.state_sum = [torch.full(c.shape, float(initial_accumulator_value), dtype=torch.float64,
                                         device=c.device) for c in self.cores]
        return self

    @property
    def tt_params(self) -> int:
        return self.shape.tt_params

    # -------------------------------------------------------------- forward
    def forward(self, input: torch.Tensor, offsets: torch.Tensor | None = None) -> torch.Tensor:
        off = to_offsets(input, offsets, self.include_last_offset)
        idx = input.reshape(-1)
        if self.allow_empty_bags and idx.numel() == 0:  # every bag empty: zero rows, zero gradients
            return torch.zeros((off.numel() - 1, self.embedding_dim), device=self.cores[0].device,
                               dtype=torch.float32) + 0.0 * sum(c.sum() for c in self.cores)
        return _TTBagFunction.apply(self, idx, off, *self.cores)

    def forward_bags(self, bags) -> torch.Tensor:
        """Reference-style batch: a list of index bags."""
        idx, off = bags_to_tensors(bags, self.cores[0].device)
        return _TTBagFunction.apply(self, idx, off, *self.cores)

    def extra_repr(self) -> str:
        return (f"{self.num_embeddings}, {self.embedding_dim}, m={self.shape.m}, n={self.shape.n}, "
                f"ranks={self.shape.ranks}")
