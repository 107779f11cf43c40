"""Config-1 bf16 query probe: time (CUDA events) and max|err| vs the oracle on a seeded
vertex subset; NDF_X3_WLO / NDF_TC_SCHEDULE select kernel variants (set before import).

    python tools/x3_probe.py [reps] [n_oracle]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_02203_b200 as ndf  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
nor = int(sys.argv[2]) if len(sys.argv) > 2 else 0
prec = os.environ.get("PREC", "bf16")
w = W.CONFIGS[1]
m = W.build_model(w, seed=0, grid_init=1.0).with_precision(prec)
ref = w.ref_position()
out = ndf.reconstruct_field_device(m, ref, ndf.ROLE_MU, w.dims)
for _ in range(3):
    ndf.reconstruct_field_device(m, ref, ndf.ROLE_MU, w.dims, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    ndf.reconstruct_field_device(m, ref, ndf.ROLE_MU, w.dims, out=out)
e1.record()
torch.cuda.synchronize()
msg = f"{prec} wlo={os.environ.get('NDF_X3_WLO', 'default')}: {e0.elapsed_time(e1) / reps:.4f} ms/query"
if nor:
    from oracle import ndf_oracle as O
    idx = np.sort(np.random.default_rng(5).choice(w.n_vertices, nor, replace=False))
    om = O.OracleModel(6, m.grid_mu, m.grid_nu, m.weights, m.biases, m.spec.merge,
                       m.spec.activation, m.spec.head_kind)
    want = O.reconstruct_field(om, ref, w.dims, vertices=idx)
    msg += f"  max|err| {np.abs(out.cpu().numpy()[idx] - want).max():.3e} ({nor} vtx)"
print(msg, flush=True)
