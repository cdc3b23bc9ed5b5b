"""Kernels of one config-1 DLRM train step (B = 256, one 1M x 16 TT field, ranks 16): python tools/cfg1_profile.py"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench_extras as bx
from paper_2507_14668_b200.model import DlrmModel, ModelConfig
dev = torch.device("cuda", 0)
torch.backends.cuda.matmul.allow_tf32 = False
cfg = ModelConfig(n_dense=6, rows_per_field=(1_000_000,), emb_dim=16, ranks=(1, 16, 16, 1), tt_threshold=1000,
                  bottom_sizes=(64,), top_sizes=(64, 32), loss="bce", seed=0)
B = 256
rng = np.random.default_rng(11)
model = DlrmModel(cfg, device=dev, max_indices=B * 3, check_errors=False, batch_size=B)
dense, sparse, labels = bx._dlrm_batch(cfg, B, rng, dev, 1, 3)
for _ in range(3):
    model.train_step(dense, sparse, labels, 0.05, 0.9, sync_loss=False)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    model.train_step(dense, sparse, labels, 0.05, 0.9, sync_loss=False)
    torch.cuda.synchronize()
ka = prof.key_averages()
print("kernels per step:", sum(k.count for k in ka), "gpu us:", sum(k.device_time_total for k in ka))
for k in sorted(ka, key=lambda k: -k.device_time_total)[:40]:
    print(f"{k.count:4d} {k.device_time_total:9.1f} us  {k.key[:90]}")
