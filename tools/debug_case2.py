import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import ttb_oracle as O
from test_gpu_parity import run_case, rel_err

g = O.Geometry((20, 20, 25), (4, 4, 4), (1, 32, 32, 1))
cores32 = [c.astype(np.float32) for c in O.init_cores(g, 3)]
c64 = [c.astype(np.float64) for c in cores32]
cases = {
    "1seg_2occ": [[0, 1]],
    "2seg_2occ": [[0, 25]],
    "2seg_3occ": [[0, 25, 1]],
    "3seg": [[30, 25, 2]],
    "pad_simple": [[7], [0, 25], [9]],
}
for name, batch in cases.items():
    idx = np.array([i for b in batch for i in b], dtype=np.int64)
    off = np.concatenate([[0], np.cumsum([len(b) for b in batch])]).astype(np.int64)
    res = run_case(g, cores32, idx, off)
    want = O.forward(c64, g, idx, off)
    print(name, rel_err(res["out"], want), np.abs(res["out"] - want).max(axis=1))
rng = np.random.default_rng(0)
for nb, L in [(64, 2), (64, 9), (64, 16), (8, 9), (8, 12), (1, 12), (1, 9), (1, 16)]:
    batch = [rng.integers(0, 1000, size=L).tolist() for _ in range(nb)]
    idx = np.array([i for b in batch for i in b], dtype=np.int64)
    off = np.concatenate([[0], np.cumsum([len(b) for b in batch])]).astype(np.int64)
    res = run_case(g, cores32, idx, off)
    want = O.forward(c64, g, idx, off)
    e = np.abs(res["out"] - want).max(axis=1)
    print(nb, L, rel_err(res["out"], want), "bad", np.nonzero(e > 1e-4)[0][:8])
