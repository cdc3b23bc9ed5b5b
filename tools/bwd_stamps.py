"""k_bwd per-phase SM cycles (TTB_DBG=8; thread 0 of block 0, averaged over
its tiles): python tools/bwd_stamps.py [cfg2|cfg3]"""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
os.environ["TTB_DBG"] = os.environ.get("TTB_DBG", "8")
from bench_extras import zipf  # noqa: E402
from paper_2507_14668_b200.engine import TtEngine  # noqa: E402
from paper_2507_14668_b200.geometry import TtShape, init_random_cores  # noqa: E402
wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
shape = TtShape((200, 200, 250), (4, 4, 4), (1, 32, 32, 1))
rng = np.random.default_rng(1)
B = 65536
pool = 1 if wl == "cfg2" else 20
T = B * pool
idx = rng.integers(0, 10_000_000, T) if wl == "cfg2" else zipf(10_000_000, T, rng)
dev = torch.device("cuda", 0)
eng = TtEngine(shape, T, B, dev)
cores = [torch.from_numpy(c).to(dev) for c in init_random_cores(shape, 0)]
ti = torch.from_numpy(idx).to(dev)
to = torch.arange(0, T + 1, pool, dtype=torch.int64, device=dev)
gout = torch.randn(B, 64, device=dev) / B
names = ["X issue + meta", "X wait", "X^T dump", "Z phase", "Z^T/image + dG2 issue", "E wait", "-",
         "reductions + next staging"]
for rep in range(3):
    eng.plan(ti, to)
    eng.forward(cores)
    eng.backward(cores, gout)
    torch.cuda.synchronize()
base = (eng._ws.data_ptr() + 255) & ~255
o = base - eng._ws.data_ptr()
h = eng._ws[o: o + 256].cpu().numpy().view(np.int64)[8:20]
nt = max(int(h[0]), 1)
tot = h[1:9].sum()
print(f"{wl}: {nt} tiles in block 0, {tot / nt:.0f} cycles per tile")
for nm, v in zip(names, h[1:9]):
    print(f"  {nm:14s} {v / nt:8.0f} cyc  {100 * v / max(tot, 1):5.1f}%")
if h[9:12].sum():
    print(f"  SIMT split (grp 0): quad setup {h[9] / nt:.0f}, lookups {h[10] / nt:.0f}, quad epilogue {h[11] / nt:.0f}")

