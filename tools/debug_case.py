import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import ttb_oracle as O
from test_gpu_parity import random_batch, run_case, rel_err

m, n, r, B, max_bag, skew = (20, 20, 25), (4, 4, 4), (1, 32, 32, 1), 500, 20, True
rng = np.random.default_rng(hash((m, B)) % 2**32)
g = O.Geometry(m, n, r)
cores32 = [c.astype(np.float32) for c in O.init_cores(g, 3)]
idx, off = random_batch(rng, g.rows, B, max_bag, skew)
gout = rng.standard_normal((B, g.cols)).astype(np.float32)
res = run_case(g, cores32, idx, off, gout)
c64 = [c.astype(np.float64) for c in cores32]
out, plan = O.forward(c64, g, idx, off, want_plan=True)
ex = res["eng"].export_plan()
print("work", np.array_equal(ex["work"], plan["work"]), "slot_occ", np.array_equal(ex["slot_occ"], plan["slot_occ"]),
      "seg_ids", np.array_equal(ex["seg_ids"], plan["seg_ids"]), "seg_inv", np.array_equal(ex["seg_inv"], plan["seg_inv"]))
err = np.abs(res["out"] - out).max(axis=1)
bad = np.nonzero(err > 1e-4)[0]
print("fwd rel", rel_err(res["out"], out), "bad bags", bad[:10], len(bad))
sizes = np.diff(off)
for b in bad[:5]:
    segs = plan["seg_inv"][off[b]:off[b+1]]
    print(b, "L", sizes[b], "S", len(set(segs.tolist())), "err", err[b])
