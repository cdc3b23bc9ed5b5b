"""TtEngine: one TT table's native handle, device workspace and call wrappers.

The engine owns no parameters; cores are passed in per call (torch CUDA
fp32 tensors in the reference layout (r_{k-1}, m_k * n_k, r_k)). All calls
are stream-ordered on torch's current stream and asynchronous, except the
status / export helpers which synchronise.

d = 2 tables run through the same d = 3 kernels with a 1x1x1 unit core in
front: geometry (m1, m2) becomes (1, m1, m2), ranks (1, R, 1) become
(1, 1, R, 1), and the two real cores keep their memory unchanged.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as nat
from .geometry import TtShape


def _ptr(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("TT-EmbeddingBag kernels need a CUDA device (no CPU fallback)")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise RuntimeError(f"TT-EmbeddingBag kernels run on CUDA devices only, got {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


class TtEngine:
    def __init__(self, shape: TtShape, max_indices: int = 1 << 16, max_bags: int | None = None, device=None,
                 deterministic: bool = False):
        """deterministic=True selects the fixed-summation-order pipeline
        (bitwise reproducible gradients, reference-ordered plan kept on the
        device). Otherwise the tensor-core pipeline runs where the geometry
        supports it (n = (4, 4, 4), ranks 32: TTB_OPT_FAST)."""
        self.shape = shape
        self.deterministic = bool(deterministic)
        self.device = require_cuda(device)
        self.lib = nat.load()
        self.is_d2 = shape.d == 2
        g = nat.TtbGeom()
        if self.is_d2:
            m, n, r = (1, *shape.m), (1, *shape.n), (1, 1, shape.ranks[1], 1)
        else:
            m, n, r = shape.m, shape.n, shape.ranks
        for k in range(3):
            g.m[k], g.n[k] = int(m[k]), int(n[k])
        for k in range(4):
            g.r[k] = int(r[k])
        self._geom = g
        self.native_m = tuple(int(v) for v in m)
        self.N = shape.cols
        self._unit = torch.ones((1, 1, 1), dtype=torch.float32, device=self.device) if self.is_d2 else None
        self._unit_grad = torch.zeros((1, 1, 1), dtype=torch.float32, device=self.device) if self.is_d2 else None
        self._handle = None
        self._ws = None
        self._sig = None
        self.max_T = 0
        self.max_B = 0
        self.plan_id = 0
        self.T = self.B = 0
        self._reserve(int(max_indices), int(max_bags if max_bags is not None else max_indices))

    # ------------------------------------------------------------ workspace
    def _reserve(self, T: int, B: int) -> None:
        T, B = max(T, 1), max(min(B, T), 1)
        nbytes = C.c_size_t()
        nat.check(self.lib.ttb_workspace_bytes(C.byref(self._geom), T, B, C.byref(nbytes)), "workspace size")
        ws = torch.empty(int(nbytes.value) + 256, dtype=torch.uint8, device=self.device)
        h = self.lib.ttb_create(C.byref(self._geom), T, B, _ptr(ws), ws.numel(), _stream())
        if not h:
            raise ValueError("ttb_create rejected the geometry / capacity")
        if self._handle:
            self.lib.ttb_destroy(self._handle)
        self._handle, self._ws = C.c_void_p(h), ws
        self.max_T, self.max_B = T, B
        if self.deterministic:
            self.set_option(nat.OPT_FAST, 0)
        if getattr(self, "_allow_empty", False):  # options live on the handle: re-apply after a resize
            self.set_option(nat.OPT_ALLOW_EMPTY, 1)

    def ensure_capacity(self, T: int, B: int) -> None:
        if T > self.max_T or B > self.max_B:
            grow = lambda need, have: max(need, int(have * 1.5))  # noqa: E731
            self._reserve(grow(T, self.max_T), grow(B, self.max_B))

    @property
    def workspace_bytes(self) -> int:
        return self._ws.numel()

    def __del__(self):
        try:
            if self._handle:
                self.lib.ttb_destroy(self._handle)
        except Exception:
            pass

    # ------------------------------------------------------------ cores
    def native_cores(self, cores):
        cores = list(cores)
        if len(cores) != self.shape.d:
            raise ValueError(f"expected {self.shape.d} cores, got {len(cores)}")
        for k, c in enumerate(cores):
            if c.device != self.device or c.dtype != torch.float32 or not c.is_contiguous():
                raise ValueError(f"core {k} must be a contiguous float32 tensor on {self.device}")
            if tuple(c.shape) != self.shape.core_extent(k):
                raise ValueError(f"core {k} extent {tuple(c.shape)} != {self.shape.core_extent(k)}")
        return [self._unit, *cores] if self.is_d2 else cores

    # ------------------------------------------------------------ calls
    def plan(self, indices: torch.Tensor, offsets: torch.Tensor) -> None:
        """indices (T,) int64/int32 CUDA; offsets (B+1,) int64 CUDA."""
        if indices.dim() != 1 or offsets.dim() != 1:
            raise ValueError("indices must be (T,), offsets (B+1,)")
        T, B = indices.numel(), offsets.numel() - 1
        if B < 1 or T < 1:
            raise ValueError("empty batch")
        if indices.dtype not in (torch.int64, torch.int32):
            raise ValueError("indices must be int64 or int32")
        if indices.device != self.device or offsets.device != self.device:
            # the kernels dereference these pointers on self.device: a host or
            # foreign-device tensor would be an illegal access, not an error
            raise ValueError(f"indices and offsets must be on {self.device}, got {indices.device} / "
                             f"{offsets.device}")
        if offsets.dtype != torch.int64:
            offsets = offsets.to(torch.int64)
        indices, offsets = indices.contiguous(), offsets.contiguous()
        self.ensure_capacity(T, B)
        nat.check(self.lib.ttb_plan(self._handle, _ptr(indices), int(indices.dtype == torch.int64), _ptr(offsets),
                                    T, B, _stream()), "plan")
        self.T, self.B = T, B
        self.plan_id += 1
        # the library may rebuild the reference-ordered plan from these later
        # (ttb_export_plan under TTB_OPT_FAST): keep them alive until the next plan
        self._plan_inputs = (indices, offsets)

    def _core_sig(self, cores):
        return tuple((c.data_ptr(), c._version) for c in cores)

    def _check_cores(self, cores) -> None:
        """The library caches derived images of the cores (ttb_cores_modified):
        drop them if any core changed through torch since the library last
        wrote or read them (torch bumps a tensor's version on every in-place
        op; the library's own fused update does not)."""
        if self._sig != self._core_sig(cores):
            nat.check(self.lib.ttb_cores_modified(self._handle), "cores_modified")

    def forward(self, cores, out: torch.Tensor | None = None) -> torch.Tensor:
        self._check_cores(cores)
        c = self.native_cores(cores)
        if out is None:
            out = torch.empty((self.B, self.N), dtype=torch.float32, device=self.device)
        nat.check(self.lib.ttb_forward(self._handle, _ptr(c[0]), _ptr(c[1]), _ptr(c[2]), _ptr(out), _stream()),
                  "forward")
        self._sig = self._core_sig(cores)
        return out

    def _gout(self, grad_out: torch.Tensor) -> torch.Tensor:
        if tuple(grad_out.shape) != (self.B, self.N):
            raise ValueError(f"grad_out must be ({self.B}, {self.N}), got {tuple(grad_out.shape)}")
        return grad_out.to(device=self.device, dtype=torch.float32).contiguous()

    def backward(self, cores, grad_out: torch.Tensor, grads=None):
        """Core gradients (list congruent to the cores)."""
        c = self.native_cores(cores)
        gout = self._gout(grad_out)
        if grads is None:
            grads = [torch.empty_like(x) for x in cores]
        g = [self._unit_grad, *grads] if self.is_d2 else list(grads)
        nat.check(self.lib.ttb_backward(self._handle, _ptr(c[0]), _ptr(c[1]), _ptr(c[2]), _ptr(gout),
                                        _ptr(g[0]), _ptr(g[1]), _ptr(g[2]), _stream()), "backward")
        return grads

    def backward_sgd(self, cores, grad_out: torch.Tensor, lr: float, momentum: float = 0.0, velocity=None):
        """Fused gradient + in-place SGD(+momentum) on the cores. velocity:
        list of fp64 tensors congruent to the cores (needed if momentum > 0)."""
        c = self.native_cores(cores)
        gout = self._gout(grad_out)
        if momentum > 0.0:
            if velocity is None or len(velocity) != self.shape.d:
                raise ValueError("momentum needs one fp64 velocity tensor per core")
            v = [None, *velocity] if self.is_d2 else list(velocity)
        else:
            v = [None, None, None]
        mask = 0b110 if self.is_d2 else 0b111
        nat.check(self.lib.ttb_backward_sgd(self._handle, _ptr(c[0]), _ptr(c[1]), _ptr(c[2]), _ptr(gout),
                                            _ptr(v[0]), _ptr(v[1]), _ptr(v[2]), float(lr), float(momentum), mask,
                                            _stream()), "backward_sgd")
        self._sig = self._core_sig(cores)

    def backward_adagrad(self, cores, grad_out: torch.Tensor, lr: float, eps: float, state_sum) -> None:
        """Gradient + in-place Adagrad on the cores (state_sum: fp64 tensors
        congruent to the cores, updated in place). Fused into the update
        kernel on the tensor-core pipeline; the deterministic pipeline returns
        its gradients and applies ttb_adagrad_update, all-or-nothing over the
        cores (every gradient is checked before any core changes)."""
        if state_sum is None or len(state_sum) != self.shape.d:
            raise ValueError("Adagrad needs one fp64 state tensor per core")
        if self.fast:
            c = self.native_cores(cores)
            s = [None, *state_sum] if self.is_d2 else list(state_sum)
            mask = 0b110 if self.is_d2 else 0b111
            nat.check(self.lib.ttb_backward_adagrad(self._handle, _ptr(c[0]), _ptr(c[1]), _ptr(c[2]),
                                                    _ptr(self._gout(grad_out)), _ptr(s[0]), _ptr(s[1]), _ptr(s[2]),
                                                    float(lr), float(eps), mask, _stream()), "backward_adagrad")
            self._sig = self._core_sig(cores)
            return
        grads = self.backward(cores, grad_out)
        err = torch.zeros(1, dtype=torch.int32, device=self.device)
        for g in grads:
            nat.check(self.lib.ttb_check_finite(_ptr(g), g.numel(), _ptr(err), _stream()), "check_finite")
        for core, g, st in zip(cores, grads, state_sum):
            nat.check(self.lib.ttb_adagrad_update(_ptr(core), _ptr(g), _ptr(st), core.numel(), float(lr), float(eps),
                                                  _ptr(err), _stream()), "adagrad_update")
        if int(err.item()):
            raise ValueError("non-finite gradient: cores and Adagrad state left unchanged")

    def aggregate(self, grad_out: torch.Tensor) -> None:
        nat.check(self.lib.ttb_aggregate(self._handle, _ptr(self._gout(grad_out)), _stream()), "aggregate")

    def allow_empty(self, on: bool = True) -> None:
        """Empty bags pool to zero rows (nn.EmbeddingBag) instead of raising."""
        self._allow_empty = bool(on)
        self.set_option(nat.OPT_ALLOW_EMPTY, int(bool(on)))

    def set_option(self, option: int, value: int) -> None:
        nat.check(self.lib.ttb_set_option(self._handle, int(option), int(value)), "set_option")

    # ------------------------------------------------------------ profiling
    def profile(self, on: bool = True) -> None:
        nat.check(self.lib.ttb_profile_enable(self._handle, int(bool(on))), "profile")

    def profile_read(self) -> dict:
        """{kernel name: (total ms, launches)} since the last read (syncs)."""
        cap = 64
        names = C.create_string_buffer(32 * cap)
        ms = (C.c_double * cap)()
        calls = (C.c_int64 * cap)()
        cnt = C.c_int()
        nat.check(self.lib.ttb_profile_read(self._handle, names, ms, calls, cap, C.byref(cnt)), "profile_read")
        raw = names.raw
        out = {}
        for i in range(cnt.value):
            nm = raw[32 * i: 32 * i + 32].split(b"\0", 1)[0].decode()
            out[nm] = (float(ms[i]), int(calls[i]))
        return out

    # ------------------------------------------------------------ read-back (sync)
    def status(self) -> dict:
        st = (C.c_int64 * 8)()
        nat.check(self.lib.ttb_read_status(self._handle, st, _stream()), "status")
        return dict(err=int(st[0]), T=int(st[1]), B=int(st[2]), P=int(st[3]), S=int(st[4]), U=int(st[5]),
                    gen=int(st[6]), items=int(st[7]))

    def plan_counts(self) -> dict:
        """S (bag-prefix segments) and U (distinct rows) of the current plan,
        counted on the device (syncs)."""
        su = (C.c_int64 * 2)()
        nat.check(self.lib.ttb_plan_counts(self._handle, su, _stream()), "plan_counts")
        return dict(S=int(su[0]), U=int(su[1]))

    def status_word(self) -> int:
        """Device address of the latched error word (ttb_status_word)."""
        return int(self.lib.ttb_status_word(self._handle))

    def check_errors(self) -> dict:
        st = self.status()
        exc = nat.errbits_to_exception(st["err"])
        if exc is not None:
            raise exc
        return st

    @property
    def fast(self) -> bool:
        """The tensor-core pipeline runs (geometry n = (4, 4, 4), ranks 32)."""
        return (not self.deterministic and not self.is_d2 and tuple(self.shape.n) == (4, 4, 4)
                and tuple(self.shape.ranks) == (1, 32, 32, 1) and self.shape.m[2] <= 288)

    def export_plan(self) -> dict:
        st = self.status()
        if st["S"] < 0:
            # tensor-core pipeline: the reference-ordered plan is built on demand
            nat.check(self.lib.ttb_export_plan(self._handle, None, None, None, None, None, _stream()), "export_plan")
            st = self.status()
        T, P, S = st["T"], st["P"], st["S"]
        dev = self.device
        work = torch.empty((max(P, 1), 4), dtype=torch.int64, device=dev)
        slot_occ = torch.empty(T, dtype=torch.int64, device=dev)
        seg_ids = torch.empty(max(S, 1), dtype=torch.int64, device=dev)
        seg_inv = torch.empty(T, dtype=torch.int64, device=dev)
        digits = torch.empty((T, 3), dtype=torch.int64, device=dev)
        nat.check(self.lib.ttb_export_plan(self._handle, _ptr(work), _ptr(slot_occ), _ptr(seg_ids), _ptr(seg_inv),
                                           _ptr(digits), _stream()), "export_plan")
        torch.cuda.current_stream().synchronize()
        out = dict(work=work[:P].cpu().numpy(), slot_occ=slot_occ.cpu().numpy(), seg_ids=seg_ids[:S].cpu().numpy(),
                   seg_inv=seg_inv.cpu().numpy(), digits=digits.cpu().numpy(), **st)
        if self.is_d2:
            out["digits"] = out["digits"][:, 1:]
        return out

    def export_fast_plan(self) -> dict:
        """The tensor-core pipeline's own plan (k_fplan output) as numpy:
        item_start (items+1), item_key (items), tile_info (tiles, 4),
        sbi (T, 2) = (bag, i3) per position, cta_tiles (CTAs+1)."""
        cnt = (C.c_int64 * 4)()
        nat.check(self.lib.ttb_export_fast_plan(self._handle, cnt, None, None, None, None, None, _stream()),
                  "export_fast_plan")
        items, tiles, ctas, T = (int(v) for v in cnt)
        dev = self.device
        bufs = dict(item_start=torch.empty(items + 1, dtype=torch.int32, device=dev),
                    item_key=torch.empty(max(items, 1), dtype=torch.int32, device=dev),
                    tile_info=torch.empty((max(tiles, 1), 4), dtype=torch.int32, device=dev),
                    sbi=torch.empty((T, 2), dtype=torch.int32, device=dev),
                    cta_tiles=torch.empty(ctas + 1, dtype=torch.int32, device=dev))
        nat.check(self.lib.ttb_export_fast_plan(self._handle, cnt, *(_ptr(bufs[k]) for k in (
            "item_start", "item_key", "tile_info", "sbi", "cta_tiles")), _stream()), "export_fast_plan")
        out = {k: v.cpu().numpy() for k, v in bufs.items()}
        out["item_key"] = out["item_key"][:items].view(np.uint32)
        out["tile_info"] = out["tile_info"][:tiles]
        out.update(items=items, tiles=tiles, ctas=ctas, T=T)
        return out

    def export_unique(self):
        st = self.status()
        U = st["U"]
        rows = torch.empty(max(U, 1), dtype=torch.int64, device=self.device)
        grads = torch.empty((max(U, 1), self.N), dtype=torch.float32, device=self.device)
        nat.check(self.lib.ttb_export_unique(self._handle, _ptr(rows), _ptr(grads), _stream()), "export_unique")
        return rows[:U], grads[:U]

    def export_slots(self) -> torch.Tensor:
        st = self.status()
        n = self.shape.n
        x = (n[0] * n[1]) if not self.is_d2 else n[0]
        r2 = self.shape.ranks[2] if not self.is_d2 else self.shape.ranks[1]
        slots = torch.empty((max(st["P"], 1), x, r2), dtype=torch.float32, device=self.device)
        nat.check(self.lib.ttb_export_slots(self._handle, _ptr(slots), _stream()), "export_slots")
        return slots[: st["P"]]


def bags_to_tensors(batch, device) -> tuple:
    """List of index bags -> (indices int64, offsets (B+1) int64) on device."""
    sizes = [len(b) for b in batch]
    flat = np.fromiter((int(i) for bag in batch for i in bag), dtype=np.int64, count=sum(sizes))
    off = np.zeros(len(batch) + 1, dtype=np.int64)
    np.cumsum(sizes, out=off[1:])
    return (torch.from_numpy(flat).to(device), torch.from_numpy(off).to(device))


def to_offsets(indices: torch.Tensor, offsets: torch.Tensor | None, include_last_offset: bool) -> torch.Tensor:
    """nn.EmbeddingBag conventions -> (B+1,) int64 offsets."""
    if indices.dim() == 2:
        B, L = indices.shape
        return torch.arange(0, B * L + 1, L, dtype=torch.int64, device=indices.device)
    if offsets is None:
        raise ValueError("1-D indices need offsets")
    offsets = offsets.to(torch.int64)
    if include_last_offset:
        return offsets
    tail = torch.full((1,), indices.numel(), dtype=torch.int64, device=offsets.device)
    return torch.cat([offsets, tail])
