"""k_bwd per-tile phase stamps (TTB_DBG=16) for block 0 at config 2."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
os.environ["TTB_DBG"] = "16"
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
gout = torch.randn(B, 64, device=dev)
names = ["c:meta", "c:staged", "c:zdone", "c:zhi", "c:p1", "c:p2", "c:end", "p:waits", "p:loads", "p:zhi", "p:zlo"]
for rep in range(2):
    eng.plan(ti, to)
    out = eng.forward(cores)
    eng.backward(cores, gout)
    torch.cuda.synchronize()
    base = (eng._ws.data_ptr() + 255) & ~255
    o = base - eng._ws.data_ptr()
    h = eng._ws[o: o + 256].cpu().numpy().view(np.uint64)[8:8 + 22].astype(np.int64).reshape(11, 2)
    t0 = h[h > 0].min()
    for nm, row in zip(names, h):
        print(f"{nm:10s}", [int(v - t0) if v else None for v in row])
    print()
