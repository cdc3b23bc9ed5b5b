import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import ttb_oracle as O
from test_gpu_parity import run_case, rel_err

g = O.Geometry((20, 20, 25), (4, 4, 4), (1, 32, 32, 1))
cores32 = [c.astype(np.float32) for c in O.init_cores(g, 3)]
c64 = [c.astype(np.float64) for c in cores32]
rng = np.random.default_rng(0)
def run(name, Ls):
    batch = [rng.integers(0, 1000, size=L).tolist() for L in Ls]
    idx = np.array([i for b in batch for i in b], dtype=np.int64)
    off = np.concatenate([[0], np.cumsum([len(b) for b in batch])]).astype(np.int64)
    res = run_case(g, cores32, idx, off)
    want = O.forward(c64, g, idx, off)
    e = np.abs(res["out"] - want).max(axis=1)
    print(name, "bad", np.nonzero(e > 1e-4)[0][:20])
run("A", [9] * 8 + [1] * 56)
run("B", [1] * 56 + [9] * 8)
run("C", [9] * 16)
run("D", [9] * 24)
run("E", [9] * 64)
run("F", [2] * 64)
run("G", [3] * 64)
run("H", [9] * 8 + [9] * 8 + [1] * 48)
