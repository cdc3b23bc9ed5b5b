"""Row-grouped backward (pooled) vs the deterministic pipeline on a Zipf
batch: python tools/rows_check.py [B] [native|permuted]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from bench_extras import zipf
from paper_2507_14668_b200.engine import TtEngine
from paper_2507_14668_b200.geometry import TtShape, init_random_cores
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
perm = len(sys.argv) > 2 and sys.argv[2] == "permuted"
shape = TtShape((200, 200, 250), (4, 4, 4), (1, 32, 32, 1))
rng = np.random.default_rng(4)
T = B * 20
idx = zipf(10_000_000, T, rng)
if perm:
    idx = np.random.default_rng(123).permutation(10_000_000)[idx]
dev = torch.device("cuda", 0)
cores = [torch.from_numpy(c).to(dev) for c in init_random_cores(shape, 0)]
ti = torch.from_numpy(idx).to(dev)
to = torch.arange(0, T + 1, 20, dtype=torch.int64, device=dev)
gout = torch.from_numpy((rng.standard_normal((B, 64)) / B).astype(np.float32)).to(dev)
res = []
for det in (False, True):
    eng = TtEngine(shape, T, B, dev, deterministic=det)
    eng.plan(ti, to)
    eng.forward(cores)
    res.append([g.clone() for g in eng.backward(cores, gout)])
    torch.cuda.synchronize()
for k in range(3):
    a, b = res[0][k].cpu().numpy(), res[1][k].cpu().numpy()
    print(k, float(np.abs(a - b).max() / np.abs(b).max()))
