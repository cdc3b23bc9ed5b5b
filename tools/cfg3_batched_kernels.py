"""Per-kernel CUDA-event times of the 26-table config-3 step through ONE
table-batched handle (as bench_extras.cfg3): python tools/cfg3_batched_kernels.py [native|permuted]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from bench_extras import zipf
from paper_2507_14668_b200.collection import BatchedTtEngine
from paper_2507_14668_b200.geometry import TtShape, init_random_cores
perm = len(sys.argv) > 1 and sys.argv[1] == "permuted"
shape = TtShape((200, 200, 250), (4, 4, 4), (1, 32, 32, 1))
tables, B, pool = 26, 65536, 20
T = B * pool
dev = torch.device("cuda", 0)
rng = np.random.default_rng(1)
idxs = []
for t in range(tables):
    ids = zipf(10_000_000, T, rng)
    if perm:
        ids = np.random.default_rng(123).permutation(10_000_000)[ids]
    idxs.append(torch.from_numpy(ids).to(dev))
beng = BatchedTtEngine([shape] * tables, B, T * tables, dev)
M = beng.M
base = init_random_cores(shape, 0)
bcores = [torch.zeros(beng.shape.core_extent(k), dtype=torch.float32, device=dev) for k in range(3)]
for t in range(tables):
    for k in range(3):
        w = shape.m[k] * shape.n[k]
        bcores[k][:, t * M[k] * shape.n[k]: t * M[k] * shape.n[k] + w, :] = torch.from_numpy(base[k]).to(dev)
bvel = [torch.zeros(c.shape, dtype=torch.float64, device=dev) for c in bcores]
bidx = torch.cat(idxs)
boff = torch.arange(0, T * tables + 1, pool, dtype=torch.int64, device=dev)
bgout = torch.randn(B, 64, device=dev).repeat(tables, 1) / B
bout = torch.empty((B * tables, 64), device=dev)
for _ in range(2):
    beng.plan(bidx, boff); beng.forward(bcores, out=bout); beng.backward_sgd(bcores, bgout, 0.05, 0.9, bvel)
torch.cuda.synchronize()
beng.profile(True); beng.profile_read()
for _ in range(3):
    beng.plan(bidx, boff); beng.forward(bcores, out=bout); beng.backward_sgd(bcores, bgout, 0.05, 0.9, bvel)
r = beng.profile_read()
tot = sum(v[0] / v[1] for v in r.values())
print("perm" if perm else "native", {k: round(v[0] / v[1], 2) for k, v in r.items()}, "ms; sum", round(tot, 2))
