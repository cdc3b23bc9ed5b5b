"""Per-kernel CUDA-event breakdown of one table step (plan + fwd + bwd + SGD)
for a chosen workload: python tools/profile_step.py [cfg2|cfg3n|cfg3p] [reps]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from bench_extras import zipf  # noqa: E402
from paper_2507_14668_b200.engine import TtEngine  # noqa: E402
from paper_2507_14668_b200.geometry import TtShape, init_random_cores  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
shape = TtShape((200, 200, 250), (4, 4, 4), (1, 32, 32, 1))
B = 65536
pool = 1 if wl == "cfg2" else 20
T = B * pool
rng = np.random.default_rng(1)
if wl == "cfg2":
    idx = rng.integers(0, 10_000_000, T)
else:
    idx = zipf(10_000_000, T, rng)
    if wl == "cfg3p":
        idx = np.random.default_rng(123).permutation(10_000_000)[idx]
dev = torch.device("cuda", 0)
eng = TtEngine(shape, T, B, dev)
cores = [torch.from_numpy(c).to(dev) for c in init_random_cores(shape, 0)]
vel = [torch.zeros(c.shape, dtype=torch.float64, device=dev) for c in cores]
ti = torch.from_numpy(idx).to(dev)
to = torch.arange(0, T + 1, pool, dtype=torch.int64, device=dev)
gout = torch.randn(B, 64, device=dev)
out = torch.empty(B, 64, device=dev)


def step():
    eng.plan(ti, to)
    eng.forward(cores, out=out)
    eng.backward_sgd(cores, gout, 0.01, 0.9, vel)


step()
torch.cuda.synchronize()
eng.profile(True)
eng.profile_read()
for _ in range(reps):
    step()
torch.cuda.synchronize()
prof = eng.profile_read()
st = eng.status()
tot = sum(ms for ms, _ in prof.values()) / reps
print(f"{wl}: T={st['T']} P={st['P']} S={st['S']} U={st['U']}  total {tot * 1e3:.1f} us/step")
for k, (ms, c) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:18s} {1e3 * ms / reps:10.1f} us  ({c // reps} launches)")
