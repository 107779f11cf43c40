"""Hang / race stress: many back-to-back grid queries on one kernel and shape.

    python tools/stress_query.py <fp16|bf16> <nx> <ny> <nz> [iterations]
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_02203_b200 as ndf  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402

prec = sys.argv[1]
dims = tuple(int(x) for x in sys.argv[2:5])
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 500
w = W.CONFIGS[1]
m = W.build_model(w, seed=0, grid_init=1.0).with_precision(prec)
ref_out = ndf.reconstruct_field_device(m, w.ref_position(), ndf.ROLE_MU, dims)
torch.cuda.synchronize()
t0 = time.time()
for i in range(iters):
    out = ndf.reconstruct_field_device(m, w.ref_position(), ndf.ROLE_MU, dims)
    if i % 50 == 49:
        torch.cuda.synchronize()
        assert torch.equal(out, ref_out), (prec, i)
        print(f"  {prec} {dims}: {i + 1} ok", flush=True)
torch.cuda.synchronize()
print(f"{prec} {dims}: {iters} queries ok in {time.time() - t0:.1f} s", flush=True)
