"""Per-phase schedule of the tcgen05 query kernel (CTA 0), from clock64 stamps.

    bash tools/build_variants.sh trace
    NDF_TC_SCHEDULE=classic NDF_TRACE_LIB=abtest/lib_trace.so python tools/trace_tc.py [--precision fp16]

(stamps are compiled only into trace builds; the classic schedule runs single-reference
queries only when NDF_TC_SCHEDULE=classic)

Events per tile: 0 start, 1 layer-0 A written, 2/4/6 hidden-layer MMA done,
3/5/7 epilogue done, 10 output MMA done.
"""

import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2307_02203_b200 as ndf  # noqa: E402
from paper_2307_02203_b200 import _native as N  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--precision", default="fp16")
    args = ap.parse_args()
    w = W.CONFIGS[1]
    model = W.build_model(w, seed=0, grid_init=1e-4).with_precision(args.precision)
    lib = N.load_library(os.environ.get("NDF_TRACE_LIB", N.LIB_PATH))
    fn = lib.ndf_debug_tc_trace
    fn.argtypes = [ctypes.c_void_p]
    buf = torch.zeros(6 * 32 * 12 + 16 + 32 * 8, dtype=torch.int64, device="cuda")
    for _ in range(3):
        ndf.reconstruct_field_device(model, w.ref_position(), ndf.ROLE_MU, w.dims)
    fn(ctypes.c_void_p(buf.data_ptr()))
    ndf.reconstruct_field_device(model, w.ref_position(), ndf.ROLE_MU, w.dims)
    torch.cuda.synchronize()
    fn(ctypes.c_void_p(0))
    allb = buf.cpu().numpy().astype(np.int64)
    ch = allb[6 * 32 * 12:].reshape(4, 4)
    print("epilogue chunks (WG0 warp0, tile 3, layer 1): start, ld done, bias st done, end")
    for c in range(4):
        print("  chunk", c, ch[c] - ch[0, 0])
    t = allb[:6 * 32 * 12].reshape(6, 32, 12)[:4]
    t0 = t[:, 0, 0].min()
    names = {0: "start", 8: "emb", 9: "bias", 11: "merge", 1: "A0", 2: "mma0", 3: "epi0",
             4: "mma1", 5: "epi1", 6: "mma2", 7: "epi2", 10: "out"}
    for wg in range(4):
        print(f"WG{wg}:")
        for k in range(3):
            row = t[wg, k]
            if row[0] == 0:
                continue
            print("  tile", k, " ".join(f"{names[e]}={row[e] - t0:>7d}" for e in names if row[e]))
    # average phase durations over tiles 2..n (steady state)
    seq = [0, 8, 9, 11, 1, 2, 3, 4, 5, 6, 7, 10]
    durs = {f"{names[a]}->{names[b]}": [] for a, b in zip(seq[:-1], seq[1:])}
    per_tile = []
    for wg in range(4):
        for k in range(2, 31):
            row = t[wg, k]
            nxt = t[wg, k + 1]
            if row[0] == 0 or nxt[0] == 0:
                continue
            for a, b in zip(seq[:-1], seq[1:]):
                durs[f"{names[a]}->{names[b]}"].append(row[b] - row[a])
            per_tile.append(nxt[0] - row[0])
    print("steady-state mean cycles per phase:")
    for k, v in durs.items():
        if v:
            print(f"  {k:12s} {np.mean(v):8.0f}")
    if per_tile:
        print(f"  tile period  {np.mean(per_tile):8.0f} cycles per WG  "
              f"({np.mean(per_tile) / 4:.0f} per tile per SM)")


if __name__ == "__main__":
    main()
