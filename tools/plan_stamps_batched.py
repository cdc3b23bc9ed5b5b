"""k_fplan phase stamps (block 0) of the 26-table batched config-3 plan: python tools/plan_stamps_batched.py [permuted]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
os.environ.setdefault("TTB_DBG", "1")
from bench_extras import zipf
from paper_2507_14668_b200.collection import BatchedTtEngine
from paper_2507_14668_b200.geometry import TtShape
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
bidx = torch.cat(idxs)
boff = torch.arange(0, T * tables + 1, pool, dtype=torch.int64, device=dev)
ws = beng._ws
for rep in range(3):
    beng.plan(bidx, boff)
    torch.cuda.synchronize()
    base = (ws.data_ptr() + 255) & ~255
    o = base - ws.data_ptr()
    h = ws[o: o + 256].cpu().numpy().view(np.uint64)[8:8 + 5].astype(np.int64)
    print("batched", "perm" if perm else "native", "phase 0 / A1 / A2 / B (us):", [round(x / 1e3, 1) for x in np.diff(h)])
