"""Tensor-core pipeline vs the deterministic pipeline (and the oracle on a
sample): python tools/check_fast.py"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from bench_extras import zipf  # noqa: E402
from oracle import ttb_oracle as O  # noqa: E402
from paper_2507_14668_b200.engine import TtEngine  # noqa: E402
from paper_2507_14668_b200.geometry import TtShape, init_random_cores  # noqa: E402


def rel(a, b):
    a = a.double().cpu()
    b = b.double().cpu()
    return float((a - b).abs().max() / max(b.abs().max(), 1e-30))


def run(name, shape, idx, off, reps=5):
    dev = torch.device("cuda", 0)
    T, B = idx.size, off.size - 1
    cores = [torch.from_numpy(c).to(dev) for c in init_random_cores(shape, 0)]
    ti, to = torch.from_numpy(idx).to(dev), torch.from_numpy(off).to(dev)
    gout = torch.randn(B, shape.cols, device=dev)
    res = {}
    for det in (True, False):
        eng = TtEngine(shape, T, B, dev, deterministic=det)
        eng.plan(ti, to)
        out = eng.forward(cores)
        st = eng.check_errors()
        grads = [g.clone() for g in eng.backward(cores, gout)]
        torch.cuda.synchronize()
        eng.profile(True)
        eng.profile_read()
        for _ in range(reps):
            eng.plan(ti, to)
            eng.forward(cores, out=torch.empty_like(out))
            eng.backward(cores, gout)
        prof = eng.profile_read()
        tot = sum(ms for ms, _ in prof.values()) / reps * 1e3
        res[det] = (out, grads, st, prof, tot)
        print(f"{name} det={det}: P={st['P']} S={st['S']} items={st['items']} kernel sum {tot:.1f} us")
        for k, (ms, c) in sorted(prof.items(), key=lambda kv: -kv[1][0])[:12]:
            print(f"    {k:18s} {1e3 * ms / reps:8.1f} us ({c // reps})")
    o1, g1 = res[True][0], res[True][1]
    o2, g2 = res[False][0], res[False][1]
    print(f"  fwd rel err fast vs det: {rel(o2, o1):.3g}")
    for k in range(3):
        print(f"  grad{k} rel err fast vs det: {rel(g2[k], g1[k]):.3g}")
    # oracle on a sample of bags (forward)
    g = O.Geometry(shape.m, shape.n, shape.ranks)
    c64 = [c.cpu().numpy().astype(np.float64) for c in cores]
    sb = np.random.default_rng(0).choice(B, min(B, 300), replace=False)
    want = np.stack([O.reconstruct_rows(c64, g, idx[off[b]:off[b + 1]]).sum(0) for b in sb])
    got = o2.cpu().numpy()[sb]
    print(f"  fwd rel err fast vs oracle (sample): {np.abs(got - want).max() / np.abs(want).max():.3g}")
    return res


if __name__ == "__main__":
    shape = TtShape((200, 200, 250), (4, 4, 4), (1, 32, 32, 1))
    rng = np.random.default_rng(1)
    B = 65536
    idx = rng.integers(0, 10_000_000, B)
    off = np.arange(B + 1, dtype=np.int64)
    run("cfg2", shape, idx, off)
    T = 65536 * 20
    idx = zipf(10_000_000, T, rng)
    off = np.arange(0, T + 1, 20, dtype=np.int64)
    run("cfg3", shape, idx, off, reps=3)
    small = TtShape((20, 20, 25), (4, 4, 4), (1, 32, 32, 1))
    sizes = rng.integers(1, 6, 3000)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    idx = rng.integers(0, 10000, int(sizes.sum()))
    run("small", small, idx, off)
