"""Per-step kernel times of the first queries in a fresh process (warm-up behaviour)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_02203_b200 as ndf  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402

w = W.CONFIGS[1]
model = W.build_model(w, seed=0, grid_init=1e-4).with_precision("fp16")
out = torch.empty(w.n_vertices, device="cuda")
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda")
ref = w.ref_position()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(40)]
for i, (a, b) in enumerate(ev):
    flush.fill_(float(i))
    a.record()
    ndf.reconstruct_field_device(model, ref, ndf.ROLE_MU, w.dims, out=out)
    b.record()
torch.cuda.synchronize()
print(" ".join(f"{a.elapsed_time(b):.3f}" for a, b in ev))
