"""Step-by-step smoke of the tensor-core pipeline (plan, forward, backward),
synchronising after each: python tools/debug_fast.py [B] [big]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2507_14668_b200.engine import TtEngine
from paper_2507_14668_b200.geometry import TtShape, init_random_cores
big = len(sys.argv) > 2
shape = TtShape((200, 200, 250) if big else (20, 20, 25), (4, 4, 4), (1, 32, 32, 1))
rng = np.random.default_rng(1)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 300
idx = rng.integers(0, shape.rows, B)
off = np.arange(B + 1, dtype=np.int64)
dev = torch.device("cuda", 0)
cores = [torch.from_numpy(c).to(dev) for c in init_random_cores(shape, 0)]
eng = TtEngine(shape, B, B, dev)
eng.plan(torch.from_numpy(idx).to(dev), torch.from_numpy(off).to(dev))
torch.cuda.synchronize(); print("plan ok", flush=True)
print(eng.status(), flush=True)
out = eng.forward(cores)
torch.cuda.synchronize(); print("fwd ok", flush=True)
g = eng.backward(cores, torch.randn(B, 64, device=dev))
torch.cuda.synchronize(); print("bwd ok", flush=True)
