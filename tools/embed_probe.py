"""Standalone positional encoder (ndf_embed_nodes) over the config-1 grid (profiling probe)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2307_02203_b200 import workloads as W  # noqa: E402

w = W.CONFIGS[1]
m = W.build_model(w, seed=0, grid_init=1.0)
for _ in range(3):
    e = m.embed_nodes("mu", w.dims)
torch.cuda.synchronize()
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0.record()
for _ in range(10):
    e = m.embed_nodes("mu", w.dims)
t1.record()
torch.cuda.synchronize()
ms = t0.elapsed_time(t1) / 10
nbytes = e.numel() * 4
print(f"embed {tuple(e.shape)}: {ms:.4f} ms, output {nbytes / ms / 1e6:.0f} GB/s written")
