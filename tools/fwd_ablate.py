"""k_fwd duration under TTB_DBG ablations (32: no epilogue math, 64: no G1 loads)."""
import os, sys, subprocess
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
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
eng.plan(ti, to); out = eng.forward(cores); torch.cuda.synchronize()
eng.profile(True); eng.profile_read()
for _ in range(20):
    eng.forward(cores, out=out)
r = eng.profile_read()
print(sys.argv[1], {k: round(v[0] / v[1] * 1e3, 1) for k, v in r.items()})
'''
for d in ["0", "32", "64", "96"]:
    env = dict(os.environ, TTB_DBG=d)
    subprocess.run([sys.executable, "-c", code, d], env=env)
