"""Reference-default architecture over the c1 grid on the exact fp32 kernel."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_02203_b200 as ndf  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402

w = W.CONFIGS[1]
V = w.n_vertices
m = ndf.NdfModel.build(ndf.ModelSpec.reference_default(), seed=0)
out = torch.empty(V, device="cuda")
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for i in range(4):
    torch.cuda.synchronize()
    t0.record()
    ndf.reconstruct_field_device(m, w.ref_position(), ndf.ROLE_MU, w.dims, out=out)
    t1.record()
    torch.cuda.synchronize()
    if i:
        ts.append(t0.elapsed_time(t1))
print(f"f3 {np.mean(ts):.3f} ms")
