"""Config-4 probe: bulk estimator pairs (Pearson + KSG) on a seeded pair list (timing only)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_02203_b200 as ndf  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
w = W.CONFIGS[4]
ens = W.generate_device(w)
ens.vertex_major()
pa, pb = W.pair_list(w, count=n, seed=2)
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ndf.pair_estimators_device(ens, "v", pa, pb, k=w.ksg_k)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{n} pairs: {dt * 1e3:.2f} ms -> {n / dt:.0f} pairs/s")
