import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2507_14668_b200.engine import TtEngine
from paper_2507_14668_b200.geometry import TtShape, init_random_cores
shape = TtShape((20, 20, 25), (4, 4, 4), (1, 32, 32, 1))
rng = np.random.default_rng(1)
sizes = rng.integers(1, 6, 3000)
off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
idx = rng.integers(0, 10000, int(sizes.sum()))
dev = torch.device("cuda", 0)
cores = [torch.from_numpy(c).to(dev) for c in init_random_cores(shape, 0)]
eng = TtEngine(shape, idx.size, 3000, dev)
ti, to = torch.from_numpy(idx).to(dev), torch.from_numpy(off).to(dev)
gout = torch.randn(3000, 64, device=dev)
for _ in range(2):
    eng.plan(ti, to); eng.forward(cores); eng.backward(cores, gout)
torch.cuda.synchronize()
