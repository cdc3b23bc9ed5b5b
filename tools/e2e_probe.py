"""e2e (host-staged) loop timing variance and raw PCIe copy bandwidth."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
from paper_2507_14668_b200.embedding_bag import TTEmbeddingBag
from paper_2507_14668_b200.staging import StagedLoop
dev = torch.device("cuda", 0)
cfg = bench.CFG2
x = torch.empty(16 << 20, dtype=torch.uint8).pin_memory()
y = torch.empty(16 << 20, dtype=torch.uint8, device=dev)
for name, f in [("h2d", lambda: y.copy_(x, non_blocking=True)), ("d2h", lambda: x.copy_(y, non_blocking=True))]:
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): f()
    b.record(); torch.cuda.synchronize()
    print(name, "GB/s", 10 * x.numel() / (a.elapsed_time(b) / 1e3) / 1e9)
emb = TTEmbeddingBag(cfg["rows"], cfg["dim"], cfg["ranks"], seed=0, max_indices=cfg["batch"], max_bags=cfg["batch"],
                     device=dev, check_errors=False).enable_fused_sgd(0.05, 0.9)
idx_h, off_h, gout_h = bench.synthetic_batch(0, cfg)
host_in = [torch.from_numpy(idx_h).pin_memory(), torch.from_numpy(off_h[:-1].copy()).pin_memory(),
           torch.from_numpy(gout_h).pin_memory()]
loop = StagedLoop(host_in, torch.empty((cfg["batch"], cfg["dim"])), dev)
def compute(i, o, g):
    out = emb(i, o)
    return out, (lambda: out.backward(g))
loop.run(compute, 3)
for rep in range(5):
    t0 = time.perf_counter()
    ms = loop.run(compute, 50)
    wall = (time.perf_counter() - t0) / 50 * 1e3
    ms_s = loop.run(compute, 50, overlap=False)
    print(f"rep {rep}: overlap {ms:.3f} ms/step (host wall {wall:.3f}), serial {ms_s:.3f}")
# host-side cost of one step without GPU waits
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    out = emb(host_in[0].to(dev, non_blocking=True), host_in[1].to(dev, non_blocking=True))
    out.backward(host_in[2].to(dev, non_blocking=True))
t1 = time.perf_counter()
torch.cuda.synchronize()
print("host issue time per step (ms)", (t1 - t0) / 50 * 1e3, "total", (time.perf_counter() - t0) / 50 * 1e3)
