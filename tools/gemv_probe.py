"""Ground-truth Pearson field on config 1 (the public path: ndf_pearson_field; profiling probe)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_02203_b200 as ndf  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402

w = W.CONFIGS[1]
ens = W.generate_device(w)
meas = ndf.CorrelationMeasure("pearson")
for _ in range(3):
    out = ndf.ground_truth_field_device(ens, meas, "v", "v", w.ref_position(), w.dims)
torch.cuda.synchronize()
print("ok", float(out[w.ref_flat()]))
