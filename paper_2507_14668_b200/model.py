"""DLRM-style model with TT-EmbeddingBag fields, on the GPU.

Mirrors the reference's model module (pkg/src/ttemb/model.py):

    ModelConfig            model.py:34-65
    loss / logit gradient  model.py:68-86   (BCE on the sigmoid, MSE)
    feature_interaction    model.py:106-112 (concat(v0, pairwise dots, lexicographic))
    Mlp                    model.py:134-173 (ReLU between, linear output)
    FieldTable             model.py:179-243 (TT above tt_threshold, dense below)
    DlrmModel              model.py:249-365 (init order, forward, train_step)
    checkpoint_bytes / save_checkpoint / load_checkpoint / read_checkpoint_records
                           model.py:388-520 (TTCKPT1 records, byte-compatible)

The TT fields run on the CUDA TT-EmbeddingBag (TTEmbeddingBag); the dense
MLPs, the interaction and the small dense fields stay in PyTorch (north star
item 4). Initialisation draws from ONE seeded numpy stream in the reference's
order, so a model built here starts from the reference's exact parameters;
train_step applies the reference's SGD(+momentum) — fp64 velocity, one
rounding into fp32 — through the library's ttb_sgd_update kernel (the TT cores
take the same step inside their backward kernels).
"""
from __future__ import annotations

import json
import math
import struct
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch
from torch import nn

from . import _native as nat
from .collection import TTEmbeddingBagCollection
from .embedding_bag import TTEmbeddingBag
from .engine import _ptr, _stream, require_cuda, to_offsets
from .geometry import bytes_to_table, factorize_dims, table_to_bytes

CKPT_MAGIC = b"TTCKPT1\n"


@dataclass(frozen=True)
class ModelConfig:
    n_dense: int
    rows_per_field: tuple
    emb_dim: int = 16
    ranks: tuple = (1, 8, 8, 1)
    tt_threshold: int = 1000
    bottom_sizes: tuple = (64,)
    top_sizes: tuple = (64, 32)
    loss: str = "bce"
    seed: int = 0

    def validate(self) -> None:
        if self.n_dense < 1 or self.emb_dim < 1 or not self.rows_per_field:
            raise ValueError("need dense features, an embedding dim, and fields")
        if any(r < 1 for r in self.rows_per_field):
            raise ValueError("every field needs at least one row")
        if self.loss not in ("bce", "mse"):
            raise ValueError(f"unknown loss {self.loss!r}")
        if self.tt_threshold < 1:
            raise ValueError("tt_threshold must be positive")
        if len(self.ranks) < 3 or self.ranks[0] != 1 or self.ranks[-1] != 1:
            raise ValueError("ranks must be (1, r_1, .., 1) with d >= 2 cores")

    @property
    def n_sparse(self) -> int:
        return len(self.rows_per_field)

    @property
    def interaction_dim(self) -> int:
        v = self.n_sparse + 1
        return self.emb_dim + v * (v - 1) // 2


def feature_interaction(vectors: Sequence[torch.Tensor]) -> torch.Tensor:
    """concat(vectors[0], all pairwise dots), pairs (0,1), (0,2), .., (1,2).."""
    stack = torch.stack(list(vectors), dim=1)  # (B, v, D)
    v = stack.shape[1]
    gram = torch.bmm(stack, stack.transpose(1, 2))
    iu = torch.triu_indices(v, v, offset=1, device=stack.device)
    # one flat column gather: its backward is an index_add along dim 1
    # (two-tensor advanced indexing would backpropagate through the much
    # slower sort-based index_put_ kernel)
    pairs = gram.reshape(gram.shape[0], v * v).index_select(1, iu[0] * v + iu[1])
    return torch.cat([vectors[0], pairs], dim=1)


class Mlp(nn.Module):
    def __init__(self, sizes: Sequence[int], rng: np.random.Generator, device):
        super().__init__()
        if len(sizes) < 2 or any(s < 1 for s in sizes):
            raise ValueError("MLP needs positive layer sizes, input to output")
        self.sizes = tuple(int(s) for s in sizes)
        last = len(sizes) - 2
        ws, bs = [], []
        for i, (fin, fout) in enumerate(zip(sizes[:-1], sizes[1:])):
            scale = math.sqrt((2.0 if i < last else 1.0) / fin)
            w = (rng.standard_normal((fin, fout)) * scale).astype(np.float32)
            ws.append(nn.Parameter(torch.from_numpy(w).to(device)))
            bs.append(nn.Parameter(torch.zeros(fout, dtype=torch.float32, device=device)))
        self.weights = nn.ParameterList(ws)
        self.biases = nn.ParameterList(bs)

    def forward(self, x):
        n = len(self.weights)
        for i in range(n):
            x = torch.addmm(self.biases[i], x, self.weights[i])
            if i < n - 1:
                x = torch.relu(x)
        return x


class _DenseBagSum(torch.autograd.Function):
    """Sum-pooled lookup of a small dense table: forward gathers rows and
    index_adds them into their bags, backward index_adds the bag gradients
    into the touched rows (atomic adds: torch's embedding_bag backward sorts
    the indices first, which dominated the DLRM step for 11 small fields)."""

    @staticmethod
    def forward(ctx, rows, indices, bag_of, n_bags):
        gathered = rows.index_select(0, indices)
        if bag_of is None:
            out = gathered
        else:
            out = torch.zeros((n_bags, rows.shape[1]), dtype=rows.dtype, device=rows.device)
            out.index_add_(0, bag_of, gathered)
        ctx.save_for_backward(indices, bag_of)
        ctx.n_rows = rows.shape[0]
        return out

    @staticmethod
    def backward(ctx, grad_out):
        indices, bag_of = ctx.saved_tensors
        g = grad_out if bag_of is None else grad_out.index_select(0, bag_of)
        grad = torch.zeros((ctx.n_rows, grad_out.shape[1]), dtype=grad_out.dtype, device=grad_out.device)
        grad.index_add_(0, indices, g.contiguous())
        return grad, None, None, None


class DenseField(nn.Module):
    """Small field below tt_threshold: plain (rows, dim) table, sum pooling."""

    def __init__(self, rows: int, dim: int, seed: int, device, check_errors: bool = True):
        super().__init__()
        self.check_errors = check_errors
        rng = np.random.default_rng(seed)
        w = (rng.standard_normal((rows, dim)) * 0.1).astype(np.float32)
        self.rows = nn.Parameter(torch.from_numpy(w).to(device))

    def forward(self, indices, offsets):
        if self.check_errors and indices.numel() and (
                int(indices.min()) < 0 or int(indices.max()) >= self.rows.shape[0]):
            raise ValueError(f"index outside [0, {self.rows.shape[0]})")
        n_bags = offsets.numel() - 1
        # bag ids from the offsets, always (the reference pools by bag id,
        # model.py:222-226: a batch with as many indices as bags may still
        # hold an empty bag next to a multi-index one); output_size avoids a
        # device->host sync
        sizes = offsets[1:] - offsets[:-1]
        bag_of = torch.repeat_interleave(torch.arange(n_bags, device=indices.device), sizes,
                                         output_size=indices.numel())
        return _DenseBagSum.apply(self.rows, indices, bag_of, n_bags)


class TTField(nn.Module):
    """A TT field served by the model's table-batched collection (its table
    f): the reference's FieldTable seam (model.py:179-243) for one field, the
    compute shared with every other TT field (one launch set per step)."""

    def __init__(self, coll: list, f: int):
        super().__init__()
        self._coll = coll  # [collection], a list so the module is registered once (as DlrmModel.tt)
        self.f = f

    @property
    def collection(self) -> TTEmbeddingBagCollection:
        return self._coll[0]

    @property
    def shape(self):
        return self.collection.shapes[self.f]

    @property
    def cores(self):
        return self.collection.table_cores(self.f)


def _tt_batchable(rows_list, emb_dim, ranks) -> bool:
    """Every TT field fits the table-batched tensor-core pipeline."""
    if len(rows_list) < 2 or tuple(ranks) != (1, 32, 32, 1):
        return False
    for rows in rows_list:
        m, n = factorize_dims(int(rows), int(emb_dim), 3)
        if tuple(n) != (4, 4, 4) or m[2] > 288:
            return False
    return True


def _is_tt(fld) -> bool:
    return isinstance(fld, (TTEmbeddingBag, TTField))


class DlrmModel(nn.Module):
    def __init__(self, config: ModelConfig, device=None, max_indices: int = 1 << 16, check_errors: bool = True,
                 batch_tt_fields: bool | None = None, batch_size: int = 1 << 12):
        """batch_tt_fields: serve every TT field from ONE table-batched
        collection (one plan / forward / backward / update launch set per step
        instead of one per field). None: whenever the fields
        fit the tensor-core pipeline (n = (4, 4, 4), ranks 32, m3 <= 288)."""
        super().__init__()
        config.validate()
        self.config = config
        dev = require_cuda(device)
        self.device = dev
        rng = np.random.default_rng(config.seed)
        seeds = [int(rng.integers(2 ** 31)) for _ in config.rows_per_field]
        tt_ids = [f for f, rows in enumerate(config.rows_per_field) if rows >= config.tt_threshold]
        if batch_tt_fields is None:
            batch_tt_fields = _tt_batchable([config.rows_per_field[f] for f in tt_ids], config.emb_dim, config.ranks)
        self.tt = None
        if batch_tt_fields and tt_ids:
            self.tt = TTEmbeddingBagCollection([(config.rows_per_field[f], config.emb_dim) for f in tt_ids],
                                               config.ranks, seeds=[seeds[f] for f in tt_ids],
                                               bags_per_table=batch_size,
                                               max_indices=max(max_indices, len(tt_ids) * batch_size),
                                               include_last_offset=True, device=dev, check_errors=check_errors)
        fields = []
        for f, rows in enumerate(config.rows_per_field):
            if rows >= config.tt_threshold:
                if self.tt is not None:
                    fields.append(TTField([self.tt], tt_ids.index(f)))
                else:
                    fields.append(TTEmbeddingBag(rows, config.emb_dim, config.ranks, seed=seeds[f], device=dev,
                                                 include_last_offset=True, max_indices=max_indices,
                                                 check_errors=check_errors))
            else:
                fields.append(DenseField(rows, config.emb_dim, seeds[f], dev, check_errors))
        self.fields = nn.ModuleList(fields)
        self.bottom = Mlp((config.n_dense, *config.bottom_sizes, config.emb_dim), rng, dev)
        self.top = Mlp((config.interaction_dim, *config.top_sizes, 1), rng, dev)
        self._velocity: dict = {}

    # ------------------------------------------------------------ parameters
    def named_ref_params(self):
        """(reference name, tensor) in DlrmModel.named_params order (model.py:272-282)."""
        out = []
        for f, fld in enumerate(self.fields):
            if _is_tt(fld):
                out.extend((f"field_{f}.core{k}", c) for k, c in enumerate(fld.cores))
            else:
                out.append((f"field_{f}.rows", fld.rows))
        for i in range(len(self.bottom.weights)):
            out.append((f"bottom.{i}.w", self.bottom.weights[i]))
            out.append((f"bottom.{i}.b", self.bottom.biases[i]))
        for i in range(len(self.top.weights)):
            out.append((f"top.{i}.w", self.top.weights[i]))
            out.append((f"top.{i}.b", self.top.biases[i]))
        return out

    def _update_params(self):
        """(name, leaf tensor) of every parameter an optimizer step touches:
        named_ref_params, with the batched TT fields' per-field core views
        replaced by the collection's stacked cores (their padding keeps zero
        gradients, so the same element-wise update leaves it zero)."""
        out = [(f"tt.core{k}", c) for k, c in enumerate(self.tt.cores)] if self.tt is not None else []
        return out + [(n, t) for n, t in self.named_ref_params()
                      if not (self.tt is not None and n.startswith("field_") and ".core" in n)]

    # ------------------------------------------------------------ forward
    def forward(self, dense: torch.Tensor, sparse) -> torch.Tensor:
        """dense (B, n_dense) fp32; sparse: per field (indices, offsets (B+1))."""
        if len(sparse) != self.config.n_sparse:
            raise ValueError("batch field count != model field count")
        v0 = self.bottom(dense)
        vectors = [v0] + [None] * len(self.fields)
        if self.tt is not None:  # every TT field in one batched lookup
            tt = [(f, sparse[f]) for f, fld in enumerate(self.fields) if isinstance(fld, TTField)]
            pooled = self._tt_lookup([s for _, s in tt]).unbind(0)  # (one stack in the backward, not F scatters)
            for j, (f, _) in enumerate(tt):
                vectors[f + 1] = pooled[j]
        for f, (fld, (idx, off)) in enumerate(zip(self.fields, sparse)):
            if not isinstance(fld, TTField):
                vectors[f + 1] = fld(idx, off)
        inter = feature_interaction(vectors)
        return self.top(inter).reshape(-1)

    def _tt_lookup(self, inputs):
        """[(indices (T_f,), offsets (B+1,))] of the TT fields -> (F, B, N):
        the fields' indices concatenated table by table, their offsets
        rebased onto one (F B + 1,) list."""
        B = inputs[0][1].numel() - 1
        if any(o.numel() - 1 != B for _, o in inputs):
            raise ValueError("every field needs the same number of bags")
        self.tt.set_bags_per_table(B)
        idx = torch.cat([i for i, _ in inputs])
        offs = torch.stack([o.to(torch.int64) for _, o in inputs])
        lens = offs[:, -1] - offs[:, 0]
        base = torch.cumsum(lens, 0) - lens - offs[:, 0]
        comb = torch.cat([(offs[:, :-1] + base[:, None]).reshape(-1), (offs[-1:, -1] + base[-1:])])
        return self.tt(idx, comb)

    def loss_and_logit_grad(self, z: torch.Tensor, y: torch.Tensor):
        """model.py:77-86: loss value (fp64) and dL/dz = (sigmoid(z) - y) / B."""
        z64, y64 = z.detach().double(), y.double()
        if self.config.loss == "bce":
            p = torch.sigmoid(z64)
            pc = p.clamp(1e-7, 1.0 - 1e-7)
            loss = -(y64 * torch.log(pc) + (1.0 - y64) * torch.log(1.0 - pc)).mean()
            gz = (p - y64) / z.numel()
        else:
            loss = ((z64 - y64) ** 2).mean()
            gz = 2.0 * (z64 - y64) / z.numel()
        return loss, gz.to(torch.float32)

    # ------------------------------------------------------------ train step
    def train_step(self, dense, sparse, labels, lr: float, momentum: float = 0.0, sync_loss: bool = True):
        """One SGD(+momentum) step over every parameter (model.py:347-365).
        TT cores are updated inside their backward kernels; everything else by
        ttb_sgd_update (fp64 velocity, one rounding)."""
        if lr < 0 or not 0.0 <= momentum < 1.0:
            raise ValueError("need lr >= 0 and 0 <= momentum < 1")
        for fld in self.fields:
            if isinstance(fld, TTEmbeddingBag):
                fld.enable_fused_sgd(lr, momentum)
        if self.tt is not None:
            self.tt.enable_fused_sgd(lr, momentum)
        for p in self.parameters():
            p.grad = None
        z = self.forward(dense, sparse)
        loss, gz = self.loss_and_logit_grad(z, labels)
        z.backward(gz)
        lib = nat.load()
        with torch.no_grad():
            # every non-core parameter in one launch (ttb_sgd_update_multi:
            # the arithmetic of ttb_sgd_update per element)
            upd, keep = [], []
            for name, p in self.named_ref_params():
                if ".core" in name:
                    continue  # TT cores: fused update already applied
                g = p.grad if p.grad is not None else torch.zeros_like(p)
                g = g.contiguous()
                v = None
                if momentum > 0.0:
                    v = self._velocity.get(name)
                    if v is None:
                        v = torch.zeros(p.shape, dtype=torch.float64, device=p.device)
                        self._velocity[name] = v
                keep.append(g)
                upd.append((p.data_ptr(), g.data_ptr(), v.data_ptr() if v is not None else None, p.numel()))
            arr = (nat.TtbSgdTensor * max(len(upd), 1))(*[nat.TtbSgdTensor(*u) for u in upd])
            nat.check(lib.ttb_sgd_update_multi(arr, len(upd), float(lr), float(momentum), _stream()), "sgd_update")
        return float(loss) if sync_loss else loss


    # ------------------------------------------------------------ data parallel
    def train_step_dp(self, dense, sparse, labels, lr: float, momentum: float = 0.0, global_batch: int | None = None,
                      group=None, sync_loss: bool = False):
        """One data-parallel SGD(+momentum) step on this rank's shard of the
        batch (Rec-AD DP; BASELINE config 5): every
        parameter's gradient — TT cores, dense fields, MLPs — lands in one
        flat fp32 buffer, scaled by local_B / global_B so the SUM over ranks
        is the gradient of the global batch mean (model.py:85-86), is
        all-reduced once, and every rank applies the same update (fp64
        velocity, one rounding), keeping the replicas identical."""
        import torch.distributed as dist
        if lr < 0 or not 0.0 <= momentum < 1.0:
            raise ValueError("need lr >= 0 and 0 <= momentum < 1")
        world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        local_b = int(labels.numel())
        global_b = int(global_batch) if global_batch is not None else local_b * world
        for fld in self.fields:
            if isinstance(fld, TTEmbeddingBag):
                fld.disable_fused_sgd()
        if self.tt is not None:
            self.tt.disable_fused_sgd()
        for p in self.parameters():
            p.grad = None
        z = self.forward(dense, sparse)
        loss, gz = self.loss_and_logit_grad(z, labels)
        z.backward(gz * (local_b / global_b))
        named = self._update_params()
        flat = torch.cat([(p.grad if p.grad is not None else torch.zeros_like(p)).reshape(-1) for _, p in named])
        if world > 1:
            dist.all_reduce(flat, group=group)
        lib = nat.load()
        off = 0
        with torch.no_grad():
            for name, p in named:
                g = flat[off:off + p.numel()]
                off += p.numel()
                v = None
                if momentum > 0.0:
                    v = self._velocity.get(name)
                    if v is None:
                        v = torch.zeros(p.shape, dtype=torch.float64, device=p.device)
                        self._velocity[name] = v
                nat.check(lib.ttb_sgd_update(_ptr(p), _ptr(g), _ptr(v), p.numel(), float(lr), float(momentum),
                                             _stream()), "sgd_update")
                p.grad = None
        return float(loss) if sync_loss else loss


def bags_field_tensors(bags_per_field, device):
    """Reference Dataset.bags (field -> sample -> bag) -> [(indices, offsets)]."""
    from .engine import bags_to_tensors
    return [bags_to_tensors(bags, device) for bags in bags_per_field]


# -------------------------------------------------------------- checkpoint
def _tensor_payload(t: torch.Tensor) -> bytes:
    """u64 ndim, u64 dims, fp32 LE data (model.py:388-391)."""
    arr = t.detach().cpu().numpy()
    head = struct.pack("<Q", arr.ndim) + b"".join(struct.pack("<Q", s) for s in arr.shape)
    return head + np.ascontiguousarray(arr, dtype="<f4").tobytes()


def _tensor_from_payload(payload: bytes, name: str) -> np.ndarray:
    if len(payload) < 8:
        raise ValueError(f"record {name}: truncated tensor header")
    ndim = struct.unpack_from("<Q", payload, 0)[0]
    if len(payload) < 8 + 8 * ndim:
        raise ValueError(f"record {name}: truncated tensor dims")
    shape = struct.unpack_from(f"<{ndim}Q", payload, 8) if ndim else ()
    body = payload[8 + 8 * ndim:]
    count = int(np.prod(shape, dtype=np.int64)) if ndim else 1
    if len(body) != 4 * count:
        raise ValueError(f"record {name}: payload size != declared shape")
    return np.frombuffer(body, dtype="<f4").reshape(shape)


def _config_payload(c: ModelConfig) -> bytes:
    doc = {"n_dense": c.n_dense, "rows_per_field": list(c.rows_per_field), "emb_dim": c.emb_dim,
           "ranks": list(c.ranks), "tt_threshold": c.tt_threshold, "bottom_sizes": list(c.bottom_sizes),
           "top_sizes": list(c.top_sizes), "loss": c.loss, "seed": c.seed}
    return json.dumps(doc, sort_keys=True, separators=(",", ":")).encode("ascii")


def _config_from_payload(payload: bytes) -> ModelConfig:
    d = json.loads(payload.decode("ascii"))
    return ModelConfig(n_dense=d["n_dense"], rows_per_field=tuple(d["rows_per_field"]), emb_dim=d["emb_dim"],
                       ranks=tuple(d["ranks"]), tt_threshold=d["tt_threshold"],
                       bottom_sizes=tuple(d["bottom_sizes"]), top_sizes=tuple(d["top_sizes"]), loss=d["loss"],
                       seed=d["seed"])


def checkpoint_bytes(model: DlrmModel) -> bytes:
    """TTCKPT1: magic, then records (u64 name len, name, u64 payload len,
    payload): config JSON, per field a TTEMB1 blob or a dense tensor, then
    the MLP tensors in named_params order (model.py:436-460)."""
    records = [("config", _config_payload(model.config))]
    for f, fld in enumerate(model.fields):
        if _is_tt(fld):
            records.append((f"field_{f}.tt", table_to_bytes(fld.shape, [c.detach().cpu().numpy()
                                                                         for c in fld.cores])))
        else:
            records.append((f"field_{f}.rows", _tensor_payload(fld.rows)))
    for name, t in model.named_ref_params():
        if not name.startswith("field_"):
            records.append((name, _tensor_payload(t)))
    out = [CKPT_MAGIC]
    for name, payload in records:
        raw = name.encode("ascii")
        out += [struct.pack("<Q", len(raw)), raw, struct.pack("<Q", len(payload)), payload]
    return b"".join(out)


def save_checkpoint(model: DlrmModel, path) -> None:
    with open(path, "wb") as fh:
        fh.write(checkpoint_bytes(model))


def parse_checkpoint(buf: bytes) -> list:
    """[(name, payload)] of a TTCKPT1 buffer (model.py:468-490)."""
    if buf[:len(CKPT_MAGIC)] != CKPT_MAGIC:
        raise ValueError("not a checkpoint file (bad magic)")
    pos, records = len(CKPT_MAGIC), []
    while pos < len(buf):
        if pos + 8 > len(buf):
            raise ValueError("truncated record header")
        (nlen,) = struct.unpack_from("<Q", buf, pos)
        pos += 8
        if pos + nlen + 8 > len(buf):
            raise ValueError("truncated record name or length")
        name = buf[pos:pos + nlen].decode("ascii")
        pos += nlen
        (size,) = struct.unpack_from("<Q", buf, pos)
        pos += 8
        if pos + size > len(buf):
            raise ValueError(f"record {name}: truncated payload")
        records.append((name, buf[pos:pos + size]))
        pos += size
    return records


def read_checkpoint_records(path) -> list:
    with open(path, "rb") as fh:
        return parse_checkpoint(fh.read())


def load_checkpoint(path, device=None, **model_kwargs) -> DlrmModel:
    """Rebuild the model from its config record, then overwrite every
    parameter from the records (model.py:493-520); strict about missing,
    mismatched and unknown records."""
    records = dict(read_checkpoint_records(path))
    if "config" not in records:
        raise ValueError("checkpoint has no config record")
    model = DlrmModel(_config_from_payload(records.pop("config")), device=device, **model_kwargs)
    with torch.no_grad():
        for f, fld in enumerate(model.fields):
            if not _is_tt(fld):
                continue
            name = f"field_{f}.tt"
            if name not in records:
                raise ValueError(f"checkpoint missing record {name}")
            shape, cores = bytes_to_table(records.pop(name))
            if shape != fld.shape:
                raise ValueError(f"record {name}: table shape mismatch")
            for dst, src in zip(fld.cores, cores):
                dst.copy_(torch.from_numpy(np.ascontiguousarray(src, dtype=np.float32)))
        for name, param in model.named_ref_params():
            if ".core" in name:
                continue
            if name not in records:
                raise ValueError(f"checkpoint missing record {name}")
            arr = _tensor_from_payload(records.pop(name), name)
            if tuple(arr.shape) != tuple(param.shape):
                raise ValueError(f"record {name}: shape mismatch")
            param.copy_(torch.from_numpy(arr.copy()))
    if records:
        raise ValueError(f"checkpoint has unknown records: {', '.join(sorted(records))}")
    return model
