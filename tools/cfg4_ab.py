"""config-4 DLRM step rate with the library named by TTB_LIB_PATH (A/B)."""
import os
import sys
import torch
sys.path.insert(0, ".")
import bench_extras as bx
r = bx.cfg4(torch.device("cuda", 0))
print(os.environ.get("TTB_LIB_PATH", "tree"), round(r["value"] / 1e6, 3), "M samples/s", round(r["ms_per_step"], 2), "ms")
