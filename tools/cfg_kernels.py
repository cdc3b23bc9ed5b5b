"""Per-kernel CUDA-event times of one table's step: python tools/cfg_kernels.py [cfg2|cfg3|cfg3p]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from bench_extras import zipf
from paper_2507_14668_b200.engine import TtEngine
from paper_2507_14668_b200.geometry import TtShape, init_random_cores
wl = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
shape = TtShape((200, 200, 250), (4, 4, 4), (1, 32, 32, 1))
rng = np.random.default_rng(1)
B = 65536
pool = 1 if wl == "cfg2" else 20
T = B * pool
idx = rng.integers(0, 10_000_000, T) if wl == "cfg2" else zipf(10_000_000, T, rng)
if wl == "cfg3p":
    idx = np.random.default_rng(123).permutation(10_000_000)[idx]
dev = torch.device("cuda", 0)
eng = TtEngine(shape, T, B, dev)
cores = [torch.from_numpy(c).to(dev) for c in init_random_cores(shape, 0)]
vel = [torch.zeros(c.shape, dtype=torch.float64, device=dev) for c in cores]
ti = torch.from_numpy(idx).to(dev)
to = torch.arange(0, T + 1, pool, dtype=torch.int64, device=dev)
gout = torch.randn(B, 64, device=dev) / B
out = torch.empty(B, 64, device=dev)
for _ in range(3):
    eng.plan(ti, to); eng.forward(cores, out=out); eng.backward_sgd(cores, gout, 0.01, 0.9, vel)
torch.cuda.synchronize()
st = eng.status()
eng.profile(True); eng.profile_read()
for _ in range(5):
    eng.plan(ti, to); eng.forward(cores, out=out); eng.backward_sgd(cores, gout, 0.01, 0.9, vel)
r = eng.profile_read()
print(wl, "P", st["P"], "items", st["items"], {k: round(v[0] / v[1] * 1e3, 1) for k, v in r.items()})
