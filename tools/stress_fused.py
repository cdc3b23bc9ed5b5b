"""Repeats the fused-SGD multi-step parity check (tests/test_gpu_parity.py::
test_fast_fused_sgd_steps_match_oracle) with varying seeds and reports the
worst errors: python tools/stress_fused.py [iterations]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import ttb_oracle as O
from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
from test_gpu_parity import random_batch, rel_err
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
worst = 0.0
for it in range(iters):
    emb = TTEmbeddingBag(10000, 64, (1, 32, 32, 1), tt_m=(20, 20, 25), tt_n=(4, 4, 4), seed=4 + it)
    emb.enable_fused_sgd(0.05, 0.9)
    g = O.Geometry(emb.shape.m, emb.shape.n, emb.shape.ranks)
    ref = [c.detach().cpu().numpy().astype(np.float32).copy() for c in emb.cores]
    vel = [None] * 3
    rng = np.random.default_rng(21 + it)
    for step in range(4):
        idx, off = random_batch(rng, 10000, 700, 4, skew=True)
        out = emb(torch.from_numpy(idx).cuda(), torch.from_numpy(off[:-1]).cuda())
        c64 = [c.astype(np.float64) for c in ref]
        fe = rel_err(out.detach().cpu().numpy(), O.forward(c64, g, idx, off))
        gout = torch.from_numpy(rng.standard_normal(out.shape).astype(np.float32)).cuda()
        out.backward(gout)
        ur, ug = O.unique_aggregate(idx, np.repeat(gout.cpu().numpy().astype(np.float64), np.diff(off), axis=0))
        want = O.core_grads(c64, g, ur, ug)
        for k in range(3):
            vel[k] = O.sgd_step(ref[k], want[k], 0.05, 0.9, vel[k])
        ce = [rel_err(emb.cores[k].detach().cpu().numpy(), ref[k]) for k in range(3)]
        if fe > 1e-5 or max(ce) > 1e-5:
            print(f"iter {it} step {step}: fwd {fe:.2e} cores {ce}", flush=True)
        worst = max(worst, fe, *ce)
print("worst", worst)
