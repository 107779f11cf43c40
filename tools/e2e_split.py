"""Where the end-to-end reconstruct_field time goes (config 1, bf16): public call wall time vs
the query kernels writing device memory / pinned host memory (CUDA events), and the host
overhead of the call around them.   python tools/e2e_split.py [reps]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_02203_b200 as ndf  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
w = W.CONFIGS[1]
m = W.build_model(w, seed=0, grid_init=1e-4).with_precision(os.environ.get("PREC", "bf16"))
ref = w.ref_position()
V = w.n_vertices
dev_out = torch.empty(V, dtype=torch.float32, device="cuda")
host_out = torch.empty(V, dtype=torch.float32, pin_memory=True)
for _ in range(20):
    ndf.reconstruct_field(m, ref, ndf.ROLE_MU, w.dims)
    ndf.reconstruct_field_device(m, ref, ndf.ROLE_MU, w.dims, out=dev_out)
    ndf.reconstruct_field_device(m, ref, ndf.ROLE_MU, w.dims, out=host_out)
torch.cuda.synchronize()


def ev_time(out):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        ndf.reconstruct_field_device(m, ref, ndf.ROLE_MU, w.dims, out=out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def wall(fn):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return 1e3 * ts[len(ts) // 2]


def one_pinned_sync():
    ndf.reconstruct_field_device(m, ref, ndf.ROLE_MU, w.dims, out=host_out)
    torch.cuda.current_stream().synchronize()


print(f"device out, back to back (events): {ev_time(dev_out):.4f} ms")
print(f"pinned out, back to back (events): {ev_time(host_out):.4f} ms")
print(f"pinned out, one call + sync (wall median): {wall(one_pinned_sync):.4f} ms")
print(f"public reconstruct_field (wall median): "
      f"{wall(lambda: ndf.reconstruct_field(m, ref, ndf.ROLE_MU, w.dims)):.4f} ms")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    torch.empty(V, dtype=torch.float32, pin_memory=True)
print(f"pinned torch.empty: {1e3 * (time.perf_counter() - t0) / reps:.4f} ms")
