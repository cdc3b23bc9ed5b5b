"""Top CUDA kernels of one config-4 TT-DLRM train step (torch.profiler / CUPTI).
   python tools/cfg4_profile.py [batched|per_field]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench_extras as bx
from paper_2507_14668_b200.model import DlrmModel, ModelConfig
dev = torch.device("cuda", 0)
torch.backends.cuda.matmul.allow_tf32 = False
cfg = ModelConfig(n_dense=13, rows_per_field=bx.KAGGLE_ROWS, emb_dim=64, ranks=(1, 32, 32, 1), tt_threshold=1000,
                  bottom_sizes=(512, 256), top_sizes=(512, 256), loss="bce", seed=0)
B = 65536
rng = np.random.default_rng(11)
mode = sys.argv[1] if len(sys.argv) > 1 else 'batched'
model = DlrmModel(cfg, device=dev, max_indices=B * 26, check_errors=False, batch_size=B,
                  batch_tt_fields=(mode == 'batched'))
dense, sparse, labels = bx._dlrm_batch(cfg, B, rng, dev, 1, 1)
for _ in range(3):
    model.train_step(dense, sparse, labels, 0.05, 0.9, sync_loss=False)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        model.train_step(dense, sparse, labels, 0.05, 0.9, sync_loss=False)
    torch.cuda.synchronize()
print(mode, 'M1..3', model.tt.engine.M if model.tt is not None else None)
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=22, max_name_column_width=50))
