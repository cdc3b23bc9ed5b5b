#!/usr/bin/env python
"""bench.py — TT-EmbeddingBag fwd+bwd(+fused SGD) throughput on B200.

Workload (BASELINE.json configs[1], the metric's single-GPU config): one TT
table of 10M rows x 64 dims, ranks (1, 32, 32, 1), m = (200, 200, 250),
n = (4, 4, 4); a step plans, forwards and back-propagates one batch of 65,536
bags of one uniform index each and applies SGD with momentum 0.9 to the
cores — the reference's forward_batch + unique_aggregate + tt_core_grads +
fused_update (pkg/src/ttemb/lookup.py:236, backward.py:72-204).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU): data parallel, weak scaling. Every rank
runs its own 65,536-lookup batch against replicated cores; core gradients are
all-reduced over NCCL (the real exchange step of Rec-AD's DP training,
PAPER.md:559-561) and every rank applies the same update.

Prints ONE JSON line on rank 0 (contract in the task statement).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CFG2 = dict(name="cfg2", rows=10_000_000, dim=64, ranks=(1, 32, 32, 1), batch=65_536, pooling=1)
LR, MU = 0.05, 0.9


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-sample", type=int, default=8192, help="lookups in the CPU-baseline sample")
    ap.add_argument("--ref-sample", type=int, default=CFG2["batch"],
                    help="lookups per reference-arm step (default: the whole config-2 batch)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip configs 1/3/4 (reported under extras)")
    ap.add_argument("--quick", action="store_true", help="skip extras (for ncu launch lists)")
    ap.add_argument("--no-graph", action="store_true", help="launch eagerly instead of replaying a CUDA graph")
    return ap.parse_args()


def synthetic_batch(rank: int, cfg=CFG2):
    """Seeded config-2 inputs: uniform indices, pooling 1."""
    rng = np.random.default_rng(1 + 1000 * rank)
    idx = rng.integers(0, cfg["rows"], cfg["batch"] * cfg["pooling"]).astype(np.int64)
    off = np.arange(0, cfg["batch"] * cfg["pooling"] + 1, cfg["pooling"], dtype=np.int64)
    # upstream gradient of a batch-mean loss: N(0, 1) / batch (keeps many
    # repeated SGD steps on one batch finite)
    gout = (np.random.default_rng(2 + 1000 * rank).standard_normal((cfg["batch"], cfg["dim"]))
            / cfg["batch"]).astype(np.float32)
    return idx, off, gout


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "10"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


# ------------------------------------------------------------------ roofline model
def algorithmic_counts(shape, T, B, P, S, U):
    n1, n2, n3 = shape.n
    r1, r2 = shape.ranks[1], shape.ranks[2]
    N, X, C = n1 * n2 * n3, n1 * n2, n2 * r2
    G = sum(math.prod(shape.core_extent(k)) for k in range(3))
    f_pre = 2 * n1 * r1 * n2 * r2
    fl = {
        "prefix_products": P * f_pre,
        "close_pool": S * 2 * X * r2 * n3 + (T - S) * r2 * n3 + (S - B) * N,
        "bwd_prefix": U * 2 * (X * r2 * n3 + r2 * n3 * X) + P * 2 * (r1 * C * n1 + n1 * r1 * C),
        "row_agg": (T - U) * N,
    }
    fwd = fl["prefix_products"] + fl["close_pool"]
    bwd = P * 2 * f_pre + U * 4 * N * r2 + (U - P) * n1 * n2 * r2 + (T - U) * N + 5 * G
    # tensor-core pipeline: whole forward / whole backward (algorithmic work
    # only: the backward's recomputation of X = G1.G2 is not counted)
    fl["f_fwd"] = fwd
    fl["f_bwd"] = bwd
    step_bytes = 2 * (T * 8 + (B + 1) * 8 + B * N * 4) + 16 * G
    return fl, fwd, bwd, step_bytes


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2507_14668_b200 import _native as nat
    from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
    from paper_2507_14668_b200.engine import _ptr, _stream

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("TTB_DIST_BACKEND", "nccl")  # gloo: several ranks on one GPU (tests)
        dist.init_process_group(backend, device_id=dev if backend == "nccl" else None)
    lib = nat.load()
    cfg = CFG2
    emb = TTEmbeddingBag(cfg["rows"], cfg["dim"], cfg["ranks"], seed=0, max_indices=cfg["batch"] * cfg["pooling"],
                         max_bags=cfg["batch"], device=dev, check_errors=False)
    shape, eng = emb.shape, emb.engine
    # flat parameter / grad / velocity buffers (cores are views) for the DP path
    from paper_2507_14668_b200 import dp
    flat = dp.FlatCores(emb.cores, device=dev)
    cores, grads, vel = flat.cores, flat.grads, flat.velocities
    flat_p, flat_g, flat_v = flat.param, flat.grad, flat.velocity

    idx_h, off_h, gout_h = synthetic_batch(rank, cfg)
    idx = torch.from_numpy(idx_h).to(dev)
    off = torch.from_numpy(off_h).to(dev)
    gout = torch.from_numpy(gout_h).to(dev)
    out = torch.empty((cfg["batch"], cfg["dim"]), dtype=torch.float32, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def local_step():
        eng.plan(idx, off)
        eng.forward(cores, out=out)
        if world == 1:
            eng.backward_sgd(cores, gout, LR, MU, vel)
        else:
            eng.backward(cores, gout, grads=grads)

    # the DP exchange step: one fused kernel per rank over peer memory
    # (reduce-scatter -> SGD of the owned shard -> all-gather, ttb_dp.cu) when
    # every GPU pair has P2P access; else NCCL all-reduce + the same update on
    # every rank (TTB_DP_EXCHANGE=nccl forces the latter)
    fused = (world > 1 and dist.get_backend() == "nccl" and os.environ.get("TTB_DP_EXCHANGE", "p2p") == "p2p"
             and dp.p2p_capable(world))
    exchange = dp.PeerExchange(flat_p, flat_g) if fused else None
    err_word = eng.status_word()

    def dp_tail():
        if exchange is not None:
            nat.check(lib.ttb_dp_exchange_update(C.byref(exchange.peers), flat_p.numel(), LR, MU, 0, _ptr(flat_v),
                                                 err_word, 0, _stream()), "dp_exchange_update")
            return
        dp.allreduce_grads(flat_g)
        nat.check(lib.ttb_sgd_update(_ptr(flat_p), _ptr(flat_g), _ptr(flat_v), flat_p.numel(), LR, MU, _stream()))

    def step():
        local_step()
        if world > 1:
            dp_tail()

    for _ in range(max(args.warmup, 3) if not args.quick else args.warmup):
        step()
    torch.cuda.synchronize()
    st = eng.check_errors()
    l0 = nat.launch_count()
    step()
    torch.cuda.synchronize()
    launches_per_step = nat.launch_count() - l0
    eager_local = local_step
    use_graph = not args.no_graph
    if use_graph:
        # the rank-local step (plan + forward + backward [+ fused update]) as
        # one CUDA graph: no host round trips between kernels; with N > 1 the
        # collective and the update follow it eagerly
        graph = torch.cuda.CUDAGraph()
        s_cap = torch.cuda.Stream()
        s_cap.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s_cap):
            local_step()
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=s_cap):
                local_step()
        torch.cuda.current_stream().wait_stream(s_cap)
        torch.cuda.synchronize()
        if world > 1 and exchange is None:
            def step():
                graph.replay()
                dp_tail()
        else:  # the fused exchange is graph-capturable: the whole DP step is one graph
            if world > 1:
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.stream(s_cap):
                    with torch.cuda.graph(graph, stream=s_cap):
                        local_step()
                        dp_tail()
                torch.cuda.current_stream().wait_stream(s_cap)
                torch.cuda.synchronize()
            step = graph.replay
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        eng.check_errors()

    clocks = ClockSampler(local).start() if not args.quick else None
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.zero_()
        evs[k][0].record()
        step()
        evs[k][1].record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = sum(a.elapsed_time(b) for a, b in evs)
    clk = clocks.stop() if clocks else None
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    lookups = cfg["batch"] * cfg["pooling"]
    value = world * lookups * args.steps / (total_ms / 1e3)

    result = {
        "metric": "TT-EmbeddingBag lookups/sec fwd+bwd", "value": value, "unit": "lookups/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded uniform indices, N(0,1)/batch upstream grads, reference init_random cores)",
        "config": {
            "workload": "BASELINE configs[1]: TT-EmbeddingBag microbench, 10M rows x 64, ranks (1,32,32,1), "
                        "m=(200,200,250) n=(4,4,4), batch 65536 bags, pooling 1, uniform indices; "
                        "step = plan + forward + backward + SGD(lr 0.05, momentum 0.9)",
            "batch_per_gpu": cfg["batch"], "pooling": cfg["pooling"],
            "parallelism": f"dp{world}" + ((" (fused P2P reduce-scatter + SGD + all-gather kernel, ttb_dp.cu)"
                                            if exchange is not None else
                                            f" ({dist.get_backend()} all-reduce of core grads + SGD)")
                                           if world > 1 else ""),
            "l2": "flushed between timed steps (512 MiB write, outside the timed events)",
            "launch": ("one CUDA graph per step" + (" + all-reduce and update" if world > 1 and exchange is None
                                                     else ""))
                      if use_graph else "eager launches",
        },
        "counts": host_counts(idx_h, off_h, shape, st),
        "pipeline": "tensor-core (TTB_OPT_FAST)" if eng.fast else "deterministic",
        "gpu_launches": int(launches_per_step * args.steps),
        "clocks": clk,
    }
    if rank == 0 and not args.quick:  # rank-local work only (no collectives)
        result.update(profile_and_roofline(args, torch, eng, lib, emb, eager_local, flush, st, dev))
    if not args.quick and not args.no_e2e:  # every rank (the DP update all-reduces)
        e2e = e2e_run(args, torch, cfg, rank, dev, world)
        if rank == 0:
            result["e2e"] = e2e
    if not args.quick and not args.no_extras:  # every rank (data-parallel DLRM, BASELINE config 5)
        import bench_extras
        cfg5 = bench_extras.cfg5(dev, world, rank)
    if rank == 0 and not args.quick:
        if world == 1 and not args.no_cpu_baseline:
            result["cpu_baseline"] = cpu_baseline(args, cfg)
        if not args.no_extras:
            pk = result.get("step_roofline", {})
            peaks = (pk["fp32_peak_tflops"], pk["hbm_gbs"]) if pk else None
            result["extras"] = bench_extras.run_all(dev, peaks, cpu=not args.no_cpu_baseline) if world == 1 else {}
            result["extras"]["cfg5_dlrm_dp"] = cfg5
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


_COUNTS = {}


def host_counts(idx_h, off_h, shape, st, cache=False):
    """T, B, P, S, U of the benchmark batch. The tensor-core pipeline does not
    form the reference's segments / unique rows, so they come from numpy."""
    if cache:
        return _COUNTS["last"]
    import numpy as np
    m3 = shape.m[-1]
    bag = np.repeat(np.arange(off_h.size - 1), np.diff(off_h))
    S = np.unique(bag.astype(np.int64) * (int(shape.rows) // m3 + 1) + idx_h // m3).size
    c = {"T": int(st["T"]), "B": int(st["B"]), "P": int(st["P"]), "S": int(S), "U": int(np.unique(idx_h).size)}
    _COUNTS["last"] = c
    return c


def profile_and_roofline(args, torch, eng, lib, emb, step, flush, st, dev):
    """Per-kernel CUDA-event durations (live, on the launch stream) over
    profiled steps; roofline of the dominant kernel and of the whole step."""
    from paper_2507_14668_b200.engine import _ptr, _stream
    nprof = max(5, min(args.steps, 20))
    eng.profile(True)
    eng.profile_read()
    for _ in range(nprof):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    prof = eng.profile_read()
    eng.profile(False)
    cnt = host_counts(None, None, emb.shape, st, cache=True)
    fl, fwd, bwd, step_bytes = algorithmic_counts(emb.shape, cnt["T"], cnt["B"], cnt["P"], cnt["S"], cnt["U"])
    kernels = {}
    for k, (ms, c) in prof.items():
        kernels[k] = {"us_per_step": 1e3 * ms / nprof, "launches_per_step": c / nprof, "avg_us": 1e3 * ms / max(c, 1)}
    dominant = max(kernels, key=lambda k: kernels[k]["us_per_step"])
    # measured FP32 FMA peak (this GPU, these clocks)
    sink = torch.zeros(256, device=dev)
    iters, blocks = 4096, 148 * 8
    best = 0.0
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        lib.ttb_fma_peak(_ptr(sink), iters, blocks, _stream())
        b.record()
        torch.cuda.synchronize()
        best = max(best, blocks * 256 * iters * 16 / (a.elapsed_time(b) / 1e3) / 1e12)
    peaks, peak_kind = measured_peaks()
    hbm = peaks["hbm_gbs"]
    step_us = sum(v["us_per_step"] for v in kernels.values())
    dk = kernels[dominant]
    traffic = None
    tp = ROOT / "profiles" / "ncu_traffic.json"
    if tp.exists():  # from one committed `ncu --set full` capture (profiles/summarize.py traffic)
        traffic = json.loads(tp.read_text())["bytes_per_launch"].get(dominant)
    if dominant in fl:
        achieved = fl[dominant] / (dk["avg_us"] * 1e-6) / 1e12
        roof = {"bound": "fp32", "kernel": dominant, "achieved": achieved, "peak": best, "unit": "TFLOP/s",
                "frac": achieved / best, "peak_source": "measured FP32 FMA probe (ttb_fma_peak) on this GPU",
                "algorithmic_flops_per_launch": fl[dominant], "traffic": traffic,
                "traffic_unit": "bytes/launch (DRAM read+write, ncu --set full, cold cache)"}
    else:
        # integer / sort kernels: bytes moved per launch (keys+values read and written)
        T = st["T"]
        U = _COUNTS["last"]["U"]
        nbytes = {"sort_rows_pass": 16 * T, "sort_rows_hist": 4 * T, "plan_mark": 8 * T + 8 * st["B"] + 12 * T,
                  "plan_slots": 8 * T, "plan_segs": 24 * T, "runs": 8 * T + 16 * U}.get(dominant, 8 * T)
        achieved = nbytes / (dk["avg_us"] * 1e-6) / 1e9
        roof = {"bound": "hbm", "kernel": dominant, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                "algorithmic_bytes_per_launch": nbytes, "traffic": traffic}
    t_flop = (fwd + bwd) / (best * 1e12)
    t_mem = step_bytes / (hbm * 1e9)
    t_roof = max(t_flop, t_mem)
    return {
        "roofline": roof,
        "step_roofline": {"flops_fwd": fwd, "flops_bwd_min": bwd, "bytes": step_bytes, "fp32_peak_tflops": best,
                          "hbm_gbs": hbm, "roofline_us": t_roof * 1e6, "kernel_sum_us": step_us,
                          "frac_of_roofline": t_roof * 1e6 / step_us,
                          "note": "SURVEY.md §8d: max(FLOPs/FP32 peak, bytes/HBM) over the kernel-time sum"},
        "kernels": {k: {kk: round(vv, 3) for kk, vv in v.items()} for k, v in sorted(kernels.items())},
    }


def e2e_run(args, torch, cfg, rank, dev, world):
    """Same metric through the public module API with HOST inputs: every
    step copies its pinned host indices / offsets / upstream grads in and its
    pooled output out, inside the timed region. Copies run on their own
    streams, double-buffered (paper_2507_14668_b200.staging): step k+1's
    inputs upload and step k's output drains while step k / k+1 compute, the
    way a production input pipeline prefetches. `serial_ms_per_step` is the
    same loop with every copy on the compute stream, for comparison. With
    N > 1 every rank runs the loop on its own batch and the backward's core
    gradients are all-reduced before the update (data parallel); the time is
    the max over ranks."""
    import torch.distributed as dist
    from paper_2507_14668_b200 import _native as nat
    from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
    from paper_2507_14668_b200.engine import _ptr, _stream
    from paper_2507_14668_b200.staging import StagedLoop
    emb = TTEmbeddingBag(cfg["rows"], cfg["dim"], cfg["ranks"], seed=0, max_indices=cfg["batch"] * cfg["pooling"],
                         max_bags=cfg["batch"], device=dev, check_errors=False)
    if world == 1:
        emb.enable_fused_sgd(LR, MU)
    else:
        lib = nat.load()
        vel = [torch.zeros(c.shape, dtype=torch.float64, device=dev) for c in emb.cores]
    idx_h, off_h, gout_h = synthetic_batch(rank, cfg)
    host_in = [torch.from_numpy(idx_h).pin_memory(),
               torch.from_numpy(off_h[:-1].copy()).pin_memory(),  # nn.EmbeddingBag-style B offsets
               torch.from_numpy(gout_h).pin_memory()]
    host_out = torch.empty((cfg["batch"], cfg["dim"]), dtype=torch.float32)

    def compute(idx_d, off_d, gout_d):
        out = emb(idx_d, off_d)
        if world == 1:
            return out, (lambda: out.backward(gout_d))

        def finish():
            out.backward(gout_d)
            flat = torch.cat([c.grad.reshape(-1) for c in emb.cores])
            dist.all_reduce(flat)
            with torch.no_grad():
                for c, g, v in zip(emb.cores, torch.split(flat, [c.numel() for c in emb.cores]), vel):
                    nat.check(lib.ttb_sgd_update(_ptr(c), _ptr(g), _ptr(v), c.numel(), LR, MU, _stream()))
                    c.grad = None
        return out, finish

    loop = StagedLoop(host_in, host_out, dev)
    steps = max(10, args.steps)
    loop.run(compute, 3)
    if world > 1:
        dist.barrier()
    ms = loop.run(compute, steps)
    if world > 1:
        dist.barrier()
    ms_serial = loop.run(compute, steps, overlap=False)
    if world > 1:
        t = torch.tensor([ms, ms_serial], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ms_serial = float(t[0]), float(t[1])
    emb.engine.check_errors()
    return {"value": world * cfg["batch"] * cfg["pooling"] / (ms / 1e3), "unit": "lookups/s", "ms_per_step": ms,
            "h2d_bytes_per_step": loop.h2d_bytes, "d2h_bytes_per_step": loop.d2h_bytes,
            "serial_ms_per_step": ms_serial,
            "path": "TTEmbeddingBag.forward + autograd backward (" + ("fused SGD" if world == 1 else
                    "core grads all-reduced, then SGD") + "); pinned host inputs in and pooled output out every "
                    "step on side copy streams (double-buffered, overlapping compute)"}


# ------------------------------------------------------------------ CPU legs (oracle port)
_W = {}


def _worker_init(cores, geom):
    _W["cores"], _W["geom"] = cores, geom


def _worker_step(args):
    """One shard of a reference step: forward_batch + unique_aggregate +
    tt_core_grads (the oracle restates lookup.py / backward.py)."""
    from oracle import ttb_oracle as O
    idx, off, gout = args
    cores, g = _W["cores"], _W["geom"]
    O.forward(cores, g, idx, off)
    rows, ug = O.unique_aggregate(idx, np.repeat(gout, np.diff(off), axis=0))
    return O.core_grads(cores, g, rows, ug)


def cpu_step_sample(cfg, n):
    from oracle import ttb_oracle as O
    g = O.Geometry((200, 200, 250), (4, 4, 4), cfg["ranks"])
    cores = [c.astype(np.float32) for c in O.init_cores(g, 0)]
    idx, off, gout = synthetic_batch(0, cfg)
    n_bags = n // cfg["pooling"]
    return g, cores, idx[: n_bags * cfg["pooling"]], off[: n_bags + 1], gout[:n_bags]


def cpu_baseline(args, cfg):
    """Oracle port (single process = 1 core for the numeric kernels) on a
    bounded sample of the same workload, on this box's host CPU."""
    from oracle import ttb_oracle as O
    g, cores, idx, off, gout = cpu_step_sample(cfg, args.cpu_sample)
    reps = 2
    t0 = time.perf_counter()
    vel = [None] * 3
    for _ in range(reps):
        _worker_init(cores, g)
        grads = _worker_step((idx, off, gout))
        for k in range(3):
            vel[k] = O.sgd_step(cores[k], grads[k], LR, MU, vel[k])
    dt = time.perf_counter() - t0
    return {"value": reps * idx.size / dt, "unit": "lookups/s", "cores": 1, "kind": "port",
            "sample": f"{reps} steps x {idx.size} lookups of the config-2 workload (oracle/ttb_oracle.py: "
                      f"forward + unique_aggregate + core_grads + sgd_step), {dt:.1f} s",
            "cpu": _cpu_model(), "host_threads_available": os.cpu_count()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args):
    """The reference arm: the reference's CPU algorithm (oracle port — the
    reference is pure numpy and cannot travel to the GPU box) on all host
    cores: each step is a bounded sample of the config-2 workload sharded over
    a process pool (core gradients are additive), then the SGD update."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp
    from oracle import ttb_oracle as O
    cfg = CFG2
    sample = min(args.ref_sample, cfg["batch"] * cfg["pooling"])
    g, cores, idx, off, gout = cpu_step_sample(cfg, sample)
    full = sample == cfg["batch"] * cfg["pooling"]
    ncores = os.cpu_count() or 1
    nw = max(1, min(ncores, sample // 256))
    bounds = np.linspace(0, gout.shape[0], nw + 1).astype(int)
    shards = []
    for a, b in zip(bounds[:-1], bounds[1:]):
        o = off[a:b + 1] - off[a]
        shards.append((idx[off[a]:off[b]], o, gout[a:b]))
    ctx = mp.get_context("fork")
    vel = [None] * 3
    with ctx.Pool(nw, initializer=_worker_init, initargs=(cores, g)) as pool:
        def step():
            parts = pool.map(_worker_step, shards)
            for k in range(3):
                tot = sum(p[k] for p in parts)
                vel[k] = O.sgd_step(cores[k], tot, LR, MU, vel[k])
        for _ in range(args.warmup):
            step()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step()
        dt = time.perf_counter() - t0
    value = args.steps * idx.size / dt
    print(json.dumps({
        "impl": "reference", "metric": "TT-EmbeddingBag lookups/sec fwd+bwd", "value": value, "unit": "lookups/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 cores, f64 gradient accumulation (reference semantics)", "data": "synthetic",
        "config": {"workload": "BASELINE configs[1]: TT-EmbeddingBag microbench, 10M rows x 64, ranks (1,32,32,1), "
                               "m=(200,200,250) n=(4,4,4), batch 65536 bags, pooling 1, uniform indices; "
                               "step = plan + forward + backward + SGD(lr 0.05, momentum 0.9)"
                               + ("" if full else f" (sample of {idx.size} lookups per step)"),
                   "batch_per_gpu": idx.size // cfg["pooling"], "pooling": cfg["pooling"],
                   "parallelism": f"{nw} CPU processes (bags sharded, core gradients summed)",
                   "same_config": full},
        "cpu_baseline": {"value": value, "unit": "lookups/s", "cores": nw, "kind": "port",
                         "sample": f"{idx.size} lookups/step sharded over {nw} processes (oracle/ttb_oracle.py)",
                         "cpu": _cpu_model()},
        "e2e": {"value": value, "unit": "lookups/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def self_launch(args) -> int:
    """`--gpus N` without a torchrun environment: re-run this command as N
    local ranks (torch.distributed.run, rendezvous on 127.0.0.1) and relay
    rank 0's JSON line, checking that it reports N GPUs."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(ROOT / "bench.py"), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the rank count is visible in the NCCL init lines (stderr)
    r = subprocess.run(cmd, stdout=subprocess.PIPE, text=True, env=env)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    if r.returncode != 0 or len(lines) != 1:
        sys.stderr.write(r.stdout)
        return r.returncode or 1
    d = json.loads(lines[0])
    if d.get("n_gpus") != args.gpus:
        sys.stderr.write(f"rank 0 reported n_gpus={d.get('n_gpus')}, expected {args.gpus}\n")
        return 1
    print(lines[0], flush=True)
    return 0


if __name__ == "__main__":
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(a))
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
