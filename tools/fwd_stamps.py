"""k_fwd per-tile phase stamps (TTB_DBG=16) for block 0 at config 2."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
os.environ.setdefault("TTB_DBG", "16")
from paper_2507_14668_b200.engine import TtEngine
from paper_2507_14668_b200.geometry import TtShape, init_random_cores
shape = TtShape((200, 200, 250), (4, 4, 4), (1, 32, 32, 1))
B = 65536
idx = np.random.default_rng(1).integers(0, shape.rows, B)
off = np.arange(B + 1, dtype=np.int64)
dev = torch.device("cuda", 0)
cores = [torch.from_numpy(c).to(dev) for c in init_random_cores(shape, 0)]
eng = TtEngine(shape, B, B, dev)
ti, to = torch.from_numpy(idx).to(dev), torch.from_numpy(off).to(dev)
for rep in range(3):
    eng.plan(ti, to)
    out = eng.forward(cores)
    torch.cuda.synchronize()
    base = (eng._ws.data_ptr() + 255) & ~255
    o = base - eng._ws.data_ptr()
    h = eng._ws[o: o + 256].cpu().numpy().view(np.uint64)[8:8 + 20].astype(np.int64).reshape(5, 4)
    t0 = h.min()
    print("rows: tile start / loads landed / MMA done / epilogue done; cols: tiles (ns)\n", h - t0)
