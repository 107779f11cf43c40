"""KSG field on a config-2 subset (profiling / timing probe)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_02203_b200 as ndf  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
w = W.CONFIGS[2]
ens = W.generate_device(w)
meas = ndf.CorrelationMeasure("ksg_mi", ksg_k=8)
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = ndf.ground_truth_field_device(ens, meas, "v", "v", w.ref_position(), w.dims, 0, n)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{n} pairs: {dt * 1e3:.2f} ms  -> {n / dt:.0f} pairs/s")
