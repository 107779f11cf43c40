"""Schedule trace of the ping-pong query kernel (query_pp_kernel), CTA 0.

E-WG rows (per tile): acc0 / epi0 / acc1 / epi1 / acc2 / epi2 / out = accumulator ready
and epilogue done times of the three hidden layers and the output stage.
P-WG rows (per fill): start, per-vertex words ready, A buffer free, layer-0 MMA issued.

Needs a trace build (stamps are compiled out of the shipped library):
    bash tools/build_variants.sh trace && NDF_TRACE_LIB=abtest/lib_trace.so python tools/trace_ws.py
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
fn = N.load_library(os.environ.get("NDF_TRACE_LIB", N.LIB_PATH)).ndf_debug_tc_trace
fn.argtypes = [ctypes.c_void_p]
buf = torch.zeros(6 * 32 * 12 + 16 + 32 * 8, dtype=torch.int64, device="cuda")
for _ in range(3):
    ndf.reconstruct_field_device(model, w.ref_position(), ndf.ROLE_MU, w.dims)
fn(ctypes.c_void_p(buf.data_ptr()))
ndf.reconstruct_field_device(model, w.ref_position(), ndf.ROLE_MU, w.dims)
torch.cuda.synchronize()
fn(ctypes.c_void_p(0))
t = buf.cpu().numpy()[:6 * 32 * 12].reshape(6, 32, 12).astype(np.int64)
t0 = t[4:6, 0, 0].min()
names = ["acc0", "epi0", "acc1", "epi1", "acc2", "epi2", "out"]
for wg in (0, 2):
    print(f"E-WG{wg} (slot {wg // 2}, columns 0-63)")
    for k in range(6):
        r = t[wg, k]
        if r[0]:
            print("  tile", k, " ".join(f"{nm}={r[e] - t0:>7d}" for e, nm in enumerate(names)))
for wg in (4, 5):
    print(f"P-WG{wg} (slot {wg - 4})")
    for k in range(6):
        r = t[wg, k]
        if r[0]:
            print("  fill", k, " ".join(f"{nm}={r[e] - t0:>7d}" for e, nm in
                                        enumerate(["start", "packed", "slot", "issued"])))
per = []
for wg in (0, 2):
    for k in range(2, 20):
        if t[wg, k + 1, 0] and t[wg, k, 0]:
            per.append(t[wg, k + 1, 0] - t[wg, k, 0])
if per:
    print(f"tile period per E-WG {np.mean(per):.0f} cycles -> {np.mean(per) / 2:.0f} per tile per SM")
e = t[[0, 2], 2:20]
for i, nm in enumerate(["acc0->epi0", "epi0->acc1", "acc1->epi1", "epi1->acc2", "acc2->epi2",
                        "epi2->out"]):
    d = (e[:, :, i + 1] - e[:, :, i])[e[:, :, 0] > 0]
    print(f"  {nm:12s} {d.mean():8.0f}")
tt = t[[0, 2]]
d = (tt[:, 3:20, 0] - tt[:, 2:19, 6])[tt[:, 3:20, 0] > 0]
print(f"  out->next acc0 {d.mean():8.0f}")

# fine events of E-WG0's layer 1 (relative to acc1): first ld done, sub-chunk 0 done,
# wait::st of K-chunk 0, K-chunk 0 barrier/issue done, wait::st of K-chunk 1, epi1
fine = []
for k in range(2, 20):
    r = t[0, k]
    if r[0] and r[7]:
        fine.append([r[7] - r[2], r[8] - r[2], r[9] - r[2], r[10] - r[2], r[11] - r[2], r[3] - r[2]])
if fine:
    f = np.mean(np.array(fine), axis=0)
    print("layer-1 fine (cycles after acc1): ld0 %.0f  sub0 %.0f  st0 %.0f  kc0 %.0f  st1 %.0f  end %.0f" % tuple(f))

# per-warp stamps of tile 3, layer 1 (E-warps 0..15): start, K-chunk 0..3 stored, end
w = buf.cpu().numpy()[6 * 32 * 12 + 16:].reshape(32, 8).astype(np.int64)
if w[0, 0]:
    base = w[:, 0].min()
    print("per-warp layer-1 stamps (tile 3), cycles after the first warp starts:")
    print("  epilogue warps: start, sub-chunk pair 0..3 stored, end")
    for i in range(16):
        print(f"  warp {i:2d} (slot {i // 8}, half {(i // 4) % 2})", " ".join(
            f"{x - base:6d}" if x else "     -" for x in w[i, [0, 1, 2, 3, 4, 6]]))
    if w[24, 0]:
        print("  issuer warps: per K-chunk barrier passed / MMAs issued")
        for i in (24, 25):
            print(f"  warp {i:2d} (slot {i - 24})        ", " ".join(
                f"{x - base:6d}" if x else "     -" for x in w[i]))
