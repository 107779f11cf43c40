"""Schedule trace of query_x3_kernel (CTA 0, both slots) from clock64 stamps.

    bash tools/build_variants.sh trace
    NDF_LIB_PATH=variants/lib_trace.so python tools/trace_x3.py
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
m = W.build_model(w, seed=0, grid_init=1e-4).with_precision(os.environ.get("PREC", "bf16"))
lib = N.load_library()
fn = lib.ndf_debug_tc_trace
fn.argtypes = [ctypes.c_void_p]
buf = torch.zeros(2 * 32 * 24, dtype=torch.int64, device="cuda")
for _ in range(3):
    ndf.reconstruct_field_device(m, w.ref_position(), ndf.ROLE_MU, w.dims)
fn(ctypes.c_void_p(buf.data_ptr()))
ndf.reconstruct_field_device(m, w.ref_position(), ndf.ROLE_MU, w.dims)
torch.cuda.synchronize()
fn(ctypes.c_void_p(0))
t = buf.cpu().numpy().reshape(2, 32, 24)
t0 = t[t > 0].min()
names = ["P:start", "P:words", "P:sfree", "P:dfree", "P:l0iss", "E:m0", "E:e0", "E:m1", "E:e1",
         "E:m2", "E:e2", "-", "I:1.0", "I:1.1", "I:1.2", "I:1.3", "I:2.0", "I:2.1", "I:2.2", "I:2.3"]
for kk in range(4, 9):
    for s in range(2):
        row = t[s, kk]
        ev = sorted((row[e] - t0, names[e]) for e in range(20) if row[e] > 0)
        print(f"slot {s} tile {kk}: " + "  ".join(f"{n}={v}" for v, n in ev))
# steady-state means (tiles 4..28)
per = {}
for s in range(2):
    for kk in range(4, 28):
        row, nxt = t[s, kk], t[s, kk + 1]
        if row[5] == 0 or nxt[5] == 0:
            continue
        seq = [(5, 6), (6, 7), (7, 8), (8, 9), (9, 10), (10, 5)]
        for a, b in seq:
            vb = nxt[b] if (a, b) == (10, 5) else row[b]
            per.setdefault(f"{names[a]}->{names[b]}", []).append(vb - row[a])
        per.setdefault("tile period", []).append(nxt[5] - row[5])
        per.setdefault("P:dfree->l0iss", []).append(row[4] - row[3])
        per.setdefault("l0iss->E:m0", []).append(row[5] - row[4])
for k, v in per.items():
    print(f"  {k:16s} {np.mean(v):8.0f} cycles")
