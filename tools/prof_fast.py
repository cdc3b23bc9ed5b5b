"""One tensor-core-pipeline step on config 2 (for ncu): python tools/prof_fast.py [cfg2|cfg3] [steps]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from bench_extras import zipf  # noqa: E402
from paper_2507_14668_b200.engine import TtEngine  # noqa: E402
from paper_2507_14668_b200.geometry import TtShape, init_random_cores  # noqa: E402
wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
shape = TtShape((200, 200, 250), (4, 4, 4), (1, 32, 32, 1))
rng = np.random.default_rng(1)
B = 65536
pool = 1 if wl == "cfg2" else 20
T = B * pool
idx = rng.integers(0, 10_000_000, T) if wl == "cfg2" else zipf(10_000_000, T, rng)
dev = torch.device("cuda", 0)
eng = TtEngine(shape, T, B, dev)
cores = [torch.from_numpy(c).to(dev) for c in init_random_cores(shape, 0)]
vel = [torch.zeros(c.shape, dtype=torch.float64, device=dev) for c in cores]
ti = torch.from_numpy(idx).to(dev)
to = torch.arange(0, T + 1, pool, dtype=torch.int64, device=dev)
gout = torch.randn(B, 64, device=dev)
out = torch.empty(B, 64, device=dev)
for _ in range(steps):
    eng.plan(ti, to)
    eng.forward(cores, out=out)
    eng.backward_sgd(cores, gout, 0.01, 0.9, vel)
torch.cuda.synchronize()
print("done", eng.status())
