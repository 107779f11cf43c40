"""Config-3 probe: 64-reference fp16 cube for both heads, PREC=bf16|fp16 MLP (timing only)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_02203_b200 as ndf  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402

w3 = W.CONFIGS[3]
V = int(np.prod(w3.dims))
refs = W.reference_vertices(w3, count=64, seed=1)
pos = np.stack([np.array([2.0 * i / (n - 1) - 1.0 for i, n in
                          zip((v % w3.dims[0], (v // w3.dims[0]) % w3.dims[1],
                               v // (w3.dims[0] * w3.dims[1])), w3.dims)]) for v in refs])
PREC = os.environ.get("PREC", "bf16")
models = [W.build_model(w3, seed=0, grid_init=1e-4).with_precision(PREC),
          ndf.NdfModel.build(ndf.ModelSpec.baseline(w3.dims, w3.latent_factor, measure_kind="ksg_mi",
                                                    precision=PREC), seed=1)]
cube = torch.empty((64, V), dtype=torch.float16, device="cuda")
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for i in range(6):
    torch.cuda.synchronize()
    t0.record()
    for m in models:
        ndf.reconstruct_multi_device(m, pos, ndf.ROLE_MU, w3.dims, 0, V, out=cube)
    t1.record()
    torch.cuda.synchronize()
    if i:
        ts.append(t0.elapsed_time(t1))
print(f"c3 {np.mean(ts):.3f} ms ({2 * 64 * V / (np.mean(ts) * 1e-3):.3e} pairs/s)")
