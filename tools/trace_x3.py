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
buf = torch.zeros(2 * 32 * 24 + 300 + 2 * 32 * 2 * 8 * 8, dtype=torch.int64, device="cuda")
for _ in range(3):
    ndf.reconstruct_field_device(m, w.ref_position(), ndf.ROLE_MU, w.dims)
fn(ctypes.c_void_p(buf.data_ptr()))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
ndf.reconstruct_field_device(m, w.ref_position(), ndf.ROLE_MU, w.dims)
e1.record()
torch.cuda.synchronize()
launch_ms = e0.elapsed_time(e1)
fn(ctypes.c_void_p(0))
tb = buf.cpu().numpy()
t = tb[:2 * 32 * 24].reshape(2, 32, 24)
cta = tb[2 * 32 * 24:2 * 32 * 24 + 296].reshape(148, 2)
c0 = tb[2 * 32 * 24 + 296:]
g0 = cta[:, 0].min()
dur = (cta[:, 1] - g0) / 1e3
print(f"CTA entry spread {(cta[:, 0].max() - g0) / 1e3:.2f} us; exit min/median/max "
      f"{dur.min():.1f}/{np.median(dur):.1f}/{dur.max():.1f} us (launch event {launch_ms * 1e3:.1f} us)")
print(f"CTA 0: {c0[1] - c0[0]} cycles in {(cta[0, 1] - cta[0, 0]) / 1e3:.1f} us -> "
      f"{(c0[1] - c0[0]) / (cta[0, 1] - cta[0, 0]):.3f} GHz")
print("slowest CTAs:", np.argsort(-dur)[:8], "fastest:", np.argsort(dur)[:8])
t0 = t[t > 0].min()
names = ["P:start", "P:words", "P:sfree", "P:dfree", "P:l0iss", "E:m0", "E:e0", "E:m1", "E:e1",
         "E:m2", "E:e2", "-", "I:1.0", "I:1.1", "I:1.2", "I:1.3", "I:2.0", "I:2.1", "I:2.2", "I:2.3", "E2:dot0", "E2:dot1", "E2:bar"]
for kk in range(4, 9):
    for s in range(2):
        row = t[s, kk]
        ev = sorted((row[e] - t0, names[e]) for e in range(23) if row[e] > 0)
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
        if row[20] > 0:
            for e in (20, 21, 22):
                per.setdefault(f"E:m2->{names[e]}", []).append(row[e] - row[9])
for k, v in per.items():
    print(f"  {k:16s} {np.mean(v):8.0f} cycles")
# implied SM clock: CTA 0's steady-state period x its tile count vs the traced launch's event time
tiles0 = -(-13750 // 148) if w.dims == (250, 352, 20) else None
if tiles0:
    est = (np.mean(per["tile period"]) * tiles0 / 2 + (t[:, 4, 5].min() - t0)) 
    print(f"  traced launch {launch_ms:.4f} ms (incl. prep); CTA-0 cycles ~{est:.0f} -> "
          f"implied clock {est / (launch_ms * 1e-3) / 1e9:.3f} GHz if CTA 0 were the critical path")

# per-warp epilogue stamps of layers 0 / 1 (relative to the lead warp's acc_full stamp)
wt = tb[2 * 32 * 24 + 300:].reshape(2, 32, 2, 8, 8)
for l in range(2):
    rel = []
    for s_ in range(2):
        for kk in range(4, 28):
            blk = wt[s_, kk, l]
            if blk[:, 0].min() <= 0:
                continue
            rel.append(blk[:, :6] - blk[0, 0])
    rel = np.mean(rel, axis=0)
    print(f"layer {l} epilogue, per warp (ch*4+wq): wait-done, ld0, arrive0..3 (cycles from lead's wait)")
    for w_ in range(8):
        print("   w%d " % w_ + " ".join(f"{v:7.0f}" for v in rel[w_]))
