"""Schedule trace of the warp-specialised query kernel (CTA 0), clock64 stamps.

E-WG rows (per item pair): A.s0..A.s3 = accumulator-ready times of slot A's stages
(3 hidden layers + output), B.* likewise, freeA/freeB = slot released.
P-WG rows (per item): start, embed done, slot acquired, layer-0 MMA issued.
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_02203_b200 as ndf  # noqa: E402
from paper_2307_02203_b200 import _native as N  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402

w = W.CONFIGS[1]
model = W.build_model(w, seed=0, grid_init=1e-4).with_precision("fp16")
fn = N.load_library().ndf_debug_tc_trace
fn.argtypes = [ctypes.c_void_p]
buf = torch.zeros(4 * 32 * 12, dtype=torch.int64, device="cuda")
for _ in range(3):
    ndf.reconstruct_field_device(model, w.ref_position(), ndf.ROLE_MU, w.dims)
fn(ctypes.c_void_p(buf.data_ptr()))
ndf.reconstruct_field_device(model, w.ref_position(), ndf.ROLE_MU, w.dims)
torch.cuda.synchronize()
fn(ctypes.c_void_p(0))
t = buf.cpu().numpy().reshape(4, 32, 12).astype(np.int64)
t0 = t[2:, 0, 0].min()
for wg in (0, 1):
    print(f"E-WG{wg}")
    for k in range(6):
        r = t[wg, k]
        if r[0] == 0:
            continue
        print("  pair", k, " ".join(f"{n}={r[e] - t0:>7d}" for n, e in
                                    [("A.s0", 0), ("A.s1", 1), ("A.s2", 2), ("A.out", 3),
                                     ("B.s0", 5), ("B.s1", 6), ("B.s2", 7), ("B.out", 8),
                                     ("freeA", 10), ("freeB", 11)] if r[e]))
for wg in (2, 3):
    print(f"P-WG{wg}")
    for k in range(8):
        r = t[wg, k]
        if r[0] == 0:
            continue
        print("  item", k, " ".join(f"{n}={r[e] - t0:>7d}" for n, e in
                                    [("start", 0), ("emb", 1), ("slot", 2), ("issued", 3)]))
# steady-state period of E-WG0 item pairs
e = t[0]
pers = [e[k + 1][0] - e[k][0] for k in range(2, 20) if e[k + 1][0] and e[k][0]]
if pers:
    print(f"E-WG0 pair period {np.mean(pers):.0f} cycles (2 tiles) -> {np.mean(pers) / 4:.0f} "
          "cycles per tile per SM")
