"""k_fplan phase stamps (block 0) at config 2 / 3: python tools/plan_stamps.py [cfg2|cfg3]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
os.environ.setdefault("TTB_DBG", "1")
from bench_extras import zipf
from paper_2507_14668_b200.engine import TtEngine
from paper_2507_14668_b200.geometry import TtShape
wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
shape = TtShape((200, 200, 250), (4, 4, 4), (1, 32, 32, 1))
B = 65536
pool = 1 if wl == "cfg2" else 20
T = B * pool
rng = np.random.default_rng(1)
idx = rng.integers(0, shape.rows, T) if wl == "cfg2" else zipf(10_000_000, T, rng)
dev = torch.device("cuda", 0)
eng = TtEngine(shape, T, B, dev)
ti, to = torch.from_numpy(idx).to(dev), torch.arange(0, T + 1, pool, dtype=torch.int64, device=dev)
for rep in range(3):
    eng.plan(ti, to)
    torch.cuda.synchronize()
    base = (eng._ws.data_ptr() + 255) & ~255
    o = base - eng._ws.data_ptr()
    h = eng._ws[o: o + 256].cpu().numpy().view(np.uint64)[8:8 + 5].astype(np.int64)
    print(wl, "phase 0 / A1 / A2 / B (ns):", list(np.diff(h)))
