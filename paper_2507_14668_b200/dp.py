"""Data-parallel TT-EmbeddingBag training (Rec-AD DP).

One process per GPU, `torch.distributed` with NCCL. TT cores are replicated;
the batch is sharded by contiguous bag ranges; every rank computes its core
gradients into ONE flat fp32 buffer, the buffer is all-reduced (SUM), and
every rank applies the same SGD(+momentum) step (fp64 velocity, one rounding:
backward.py:186-204), so replicas stay bitwise identical.

The host-side pieces (sharding, flat buffers, the all-reduce) are plain
torch and are exercised on CPU with the gloo backend (tests/test_dp.py); the
compute runs through TtEngine (CUDA only).
"""
from __future__ import annotations

import ctypes as C
import math

import torch
import torch.distributed as dist


def shard_bags(offsets: torch.Tensor, rank: int, world: int):
    """Contiguous bag range [b0, b1) of `rank` and its index range [t0, t1)
    for (B+1)-style offsets. Bags are split as evenly as possible."""
    B = offsets.numel() - 1
    b0 = (B * rank) // world
    b1 = (B * (rank + 1)) // world
    t0, t1 = int(offsets[b0]), int(offsets[b1])
    return b0, b1, t0, t1


def local_batch(indices: torch.Tensor, offsets: torch.Tensor, rank: int, world: int):
    """This rank's (indices, offsets) slice, offsets rebased to 0."""
    b0, b1, t0, t1 = shard_bags(offsets, rank, world)
    return indices[t0:t1], offsets[b0:b1 + 1] - offsets[b0], (b0, b1)


class FlatCores:
    """Flat fp32 parameter and gradient buffers and an fp64 velocity buffer,
    with per-core views in the reference layout (r_{k-1}, m_k n_k, r_k)."""

    def __init__(self, cores, device=None):
        cores = [c.detach() for c in cores]
        dev = device if device is not None else cores[0].device
        self.shapes = [tuple(c.shape) for c in cores]
        self.sizes = [math.prod(s) for s in self.shapes]
        self.param = torch.cat([c.reshape(-1).to(dev, torch.float32) for c in cores]).contiguous()
        self.grad = torch.zeros_like(self.param)
        self.velocity = torch.zeros(self.param.numel(), dtype=torch.float64, device=dev)

    def _views(self, flat):
        return [v.view(s) for v, s in zip(torch.split(flat, self.sizes), self.shapes)]

    @property
    def cores(self):
        return self._views(self.param)

    @property
    def grads(self):
        return self._views(self.grad)

    @property
    def velocities(self):
        return self._views(self.velocity)


def allreduce_grads(flat_grad: torch.Tensor, group=None, scale: float | None = None) -> torch.Tensor:
    """SUM all-reduce of the flat gradient buffer (in place). `scale` (e.g.
    local_B / global_B for a batch-mean loss, model.py:85-86) is applied on
    the local contribution before the reduction."""
    if scale is not None and scale != 1.0:
        flat_grad.mul_(scale)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(flat_grad, op=dist.ReduceOp.SUM, group=group)
    return flat_grad


def dp_step(engine, flat: FlatCores, indices, offsets, grad_out, lr: float, momentum: float = 0.0, group=None):
    """One data-parallel step on this rank's shard: plan, forward (returned),
    core gradients, all-reduce, SGD(+momentum) on the flat buffers."""
    from . import _native as nat
    from .engine import _ptr, _stream

    engine.plan(indices, offsets)
    out = engine.forward(flat.cores)
    engine.backward(flat.cores, grad_out, grads=flat.grads)
    allreduce_grads(flat.grad, group)
    checked_update(flat.param, flat.grad, flat.velocity if momentum > 0 else None, lr, momentum)
    return out


def checked_update(param: torch.Tensor, grad: torch.Tensor, velocity, lr: float, momentum: float,
                   err: torch.Tensor | None = None, raise_now: bool = True) -> torch.Tensor:
    """fused_update semantics (backward.py:186-204) on a flat buffer: the
    gradient is checked for non-finite values on the device first and the
    update is skipped (param and velocity untouched) if any is found.
    `err` (one int32 on the device) accumulates the error bits; with
    raise_now the call syncs and raises ValueError like the reference."""
    from . import _native as nat
    from .engine import _ptr, _stream

    if err is None:
        err = torch.zeros(1, dtype=torch.int32, device=param.device)
    lib = nat.load()
    nat.check(lib.ttb_sgd_update_checked(_ptr(param), _ptr(grad), _ptr(velocity) if momentum > 0 else None,
                                         param.numel(), float(lr), float(momentum), _ptr(err), _stream()),
              "sgd_update_checked")
    if raise_now:
        exc = nat.errbits_to_exception(int(err.item()))
        if exc is not None:
            raise exc
    return err


# ------------------------------------------------------------------ fused exchange over peer memory
class PeerExchange:
    """The data-parallel exchange step as ONE kernel per rank over peer
    memory (ttb_dp_exchange_update, csrc/ttb_dp.cu): reduce-scatter of the
    flat gradient buffers, the optimizer update of this rank's shard, and
    all-gather of the new parameters by P2P stores — instead of an NCCL
    all-reduce followed by the same update on every rank.

    Ranks in separate processes (one GPU each) map each other's flat
    param / grad buffers and flag words through CUDA IPC; the handles travel
    over the process group (all_gather_object). `flat_param` / `flat_grad`
    must stay allocated (and at the same address) for the object's life."""

    def __init__(self, flat_param: torch.Tensor, flat_grad: torch.Tensor, group=None, grid: int = 0):
        from . import _native as nat
        from .engine import _ptr
        self.lib = nat.load()
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        if self.world > nat.DP_MAX_PEERS:
            raise ValueError(f"at most {nat.DP_MAX_PEERS} ranks")
        if flat_param.numel() != flat_grad.numel():
            raise ValueError("param and grad buffers differ in length")
        self.n = flat_param.numel()
        self.grid = int(grid)
        self.flags = torch.zeros(int(self.lib.ttb_dp_flag_words(self.world)), dtype=torch.int32,
                                 device=flat_param.device)
        self._keep = (flat_param, flat_grad, self.flags)
        self._opened = []
        mine = [_ptr(flat_grad), _ptr(flat_param), _ptr(self.flags)]
        if self.world == 1:
            table = [mine]
        else:
            shared = []
            for p in mine:
                h = (C.c_char * 64)()
                off = C.c_int64(0)
                nat.check(self.lib.ttb_ipc_handle(p, h, C.byref(off)), "ipc_handle")
                shared.append((bytes(h), int(off.value)))
            allh = [None] * self.world
            dist.all_gather_object(allh, shared, group=group)
            torch.cuda.synchronize()
            table = []
            for r, entries in enumerate(allh):
                if r == self.rank:
                    table.append(mine)
                    continue
                ptrs, bases = [], {}
                for h, off in entries:  # buffers may share one allocation: map each handle once
                    if h not in bases:
                        out = C.c_void_p()
                        nat.check(self.lib.ttb_ipc_open(C.c_char_p(h), 0, C.byref(out)), "ipc_open")
                        self._opened.append((out.value, 0))
                        bases[h] = out.value
                    ptrs.append(bases[h] + off)
                table.append(ptrs)
        self.peers = make_peers(self.rank, table)

    def step(self, lr: float, momentum: float = 0.0, state: torch.Tensor | None = None, err=None,
             adagrad: bool = False, eps: float = 1e-10):
        """One exchange + update. state: fp64, length n (velocity, or Adagrad
        sums); err: device int32 — non-zero on entry (e.g. a failed local
        finiteness check) cancels the update on EVERY rank."""
        from . import _native as nat
        from .engine import _ptr, _stream
        nat.check(self.lib.ttb_dp_exchange_update(C.byref(self.peers), self.n, float(lr),
                                                  float(eps if adagrad else momentum), int(adagrad),
                                                  _ptr(state) if state is not None else None,
                                                  _ptr(err) if err is not None else None, self.grid, _stream()),
                  "dp_exchange_update")

    def close(self):
        for p, off in self._opened:
            self.lib.ttb_ipc_close(p, off)
        self._opened = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def make_peers(rank: int, table):
    """ttb_dp_peers from [(grad_ptr, param_ptr, flags_ptr)] per rank."""
    from . import _native as nat
    P = nat.DpPeers()
    P.rank, P.world = rank, len(table)
    for r, (g, p, f) in enumerate(table):
        P.grad[r], P.param[r], P.flags[r] = g, p, f
    return P


def p2p_capable(world: int) -> bool:
    """Every pair of the node's first `world` GPUs can access each other
    (the fused exchange needs peer loads / stores)."""
    if world < 2 or torch.cuda.device_count() < world:
        return False
    return all(torch.cuda.can_device_access_peer(a, b) for a in range(world) for b in range(world) if a != b)
