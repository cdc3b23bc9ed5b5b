"""Host <-> device staging for training / serving loops over host batches.

A step of the TT-EmbeddingBag path consumes host-resident batches (indices,
offsets and, in the microbenchmark, the upstream gradient) and produces a
host-visible result (the pooled output or a loss). Issuing those copies on
the compute stream serialises PCIe with the kernels; StagedLoop puts uploads
and downloads on their own streams with `depth` device slots, so step k+1's
inputs upload and step k's result drains while the GPU computes — every
step's bytes still cross PCIe inside the loop.

The reference has no device and therefore no equivalent; its loop is
DlrmModel.train_step over numpy batches (model.py:347-365).
"""
from __future__ import annotations

from typing import Callable, Sequence

import torch


class StagedLoop:
    """Double-buffered host->device inputs and device->host results.

    host_in: list of host tensors (pinned here if they are not), or a callable
    k -> list of host tensors of the same shapes (one batch per step).
    host_out: a host tensor shaped like the per-step result.
    """

    def __init__(self, host_in, host_out: torch.Tensor, device, depth: int = 2):
        self.device = torch.device(device)
        self.depth = int(depth)
        if callable(host_in):
            self._host_fn = host_in
            proto = host_in(0)
        else:
            pinned = [h if h.is_pinned() else h.pin_memory() for h in host_in]
            self._host_fn = lambda k: pinned
            proto = pinned
        self.dev_in = [[torch.empty(h.shape, dtype=h.dtype, device=self.device) for h in proto]
                       for _ in range(self.depth)]
        self.host_out = [torch.empty(host_out.shape, dtype=host_out.dtype).pin_memory() for _ in range(self.depth)]
        self.out_ready = [torch.cuda.Event() for _ in range(self.depth)]
        self.h2d_stream = torch.cuda.Stream(self.device)
        self.d2h_stream = torch.cuda.Stream(self.device)
        self.h2d_bytes = int(sum(h.numel() * h.element_size() for h in proto))
        self.d2h_bytes = int(host_out.numel() * host_out.element_size())

    def run(self, compute: Callable[..., tuple], steps: int, overlap: bool = True) -> float:
        """Run `steps` steps; returns device-timed ms per step (first upload
        to last download). compute(*device_inputs) -> (result, finish):
        `result` is copied to the host as soon as it is produced, then
        finish() runs the rest of the step (e.g. the backward)."""
        cur = torch.cuda.current_stream(self.device)
        D = self.depth
        h2d = self.h2d_stream if overlap else cur
        d2h = self.d2h_stream if overlap else cur
        ev_in = [torch.cuda.Event() for _ in range(D)]
        ev_free: list = [None] * D
        ev_out = [torch.cuda.Event() for _ in range(D)]
        # each result stays referenced until the compute stream has waited for
        # its download (instead of record_stream, whose deferred frees make the
        # caching allocator fall back to fresh cudaMallocs under this pattern)
        hold: list = [None] * D
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(self.device)
        start.record(cur)
        if overlap:
            h2d.wait_event(start)

        def upload(k: int) -> None:
            s = k % D
            if ev_free[s] is not None:
                h2d.wait_event(ev_free[s])
            with torch.cuda.stream(h2d):
                for d, h in zip(self.dev_in[s], self._host_fn(k)):
                    d.copy_(h, non_blocking=True)
            ev_in[s].record(h2d)

        if overlap:
            for k in range(min(D, steps)):
                upload(k)
        for k in range(steps):
            s = k % D
            if not overlap:
                upload(k)
            cur.wait_event(ev_in[s])
            if hold[s] is not None:
                cur.wait_event(ev_out[s])
                hold[s] = None
            result, finish = compute(*self.dev_in[s])
            ev = torch.cuda.Event()
            ev.record(cur)
            d2h.wait_event(ev)
            with torch.cuda.stream(d2h):
                self.host_out[s].copy_(result.detach(), non_blocking=True)
            self.out_ready[s].record(d2h)
            ev_out[s].record(d2h)
            hold[s] = result
            if finish is not None:
                finish()
            fr = torch.cuda.Event()
            fr.record(cur)
            ev_free[s] = fr
            if overlap and k + D < steps:
                upload(k + D)
        cur.wait_stream(d2h)
        end.record(cur)
        torch.cuda.synchronize(self.device)
        return start.elapsed_time(end) / max(steps, 1)

    def result(self, k: int) -> torch.Tensor:
        """Host copy of step k's result (waits for its download)."""
        s = k % self.depth
        self.out_ready[s].synchronize()
        return self.host_out[s]


def stage_batches(batches: Sequence[Sequence[torch.Tensor]]):
    """Callable k -> pinned host tensors cycling over `batches`."""
    pinned = [[t if t.is_pinned() else t.pin_memory() for t in b] for b in batches]
    return lambda k: pinned[k % len(pinned)]
