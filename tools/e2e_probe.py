"""Break down the end-to-end reconstruct_field latency (host wall clock)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_02203_b200 as ndf  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402

w = W.CONFIGS[1]
model = W.build_model(w, seed=0, grid_init=1e-4).with_precision("fp16")
ref = w.ref_position()
V = w.n_vertices


def t(fn, n=30):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e3 * np.median(ts)


out = torch.empty(V, device="cuda")
host = torch.empty(V, pin_memory=True)
print("device query only      %.3f ms" % t(lambda: ndf.reconstruct_field_device(model, ref, ndf.ROLE_MU, w.dims, out=out)))
print("D2H 7 MB pinned        %.3f ms" % t(lambda: host.copy_(out, non_blocking=True)))
print("D2H 7 MB pageable      %.3f ms" % t(lambda: out.cpu()))
print("pinned alloc 7 MB      %.3f ms" % t(lambda: torch.empty(V, pin_memory=True)))
print("query + pinned D2H     %.3f ms" % t(lambda: host.copy_(ndf.reconstruct_field_device(model, ref, ndf.ROLE_MU, w.dims, out=out), non_blocking=True)))
print("reconstruct_field      %.3f ms" % t(lambda: ndf.reconstruct_field(model, ref, ndf.ROLE_MU, w.dims)))
print("np.empty 7MB + memcpy  %.3f ms" % t(lambda: np.copy(host.numpy())))
print("query into pinned host  %.3f ms" % t(lambda: ndf.reconstruct_field_device(model, ref, ndf.ROLE_MU, w.dims, out=host)))
st = model.device_state()
from paper_2307_02203_b200 import _native as N  # noqa: E402
from paper_2307_02203_b200.model import ctypes_ref  # noqa: E402
desc = ctypes_ref(st.desc)
stream = N.stream_handle(st.device)
prec = N.PREC["fp16"]
lib = N.load_library()
hp = host.data_ptr()
print("raw C-ABI into pinned   %.3f ms" % t(lambda: lib.ndf_query_grid(desc, float(ref[0]), float(ref[1]), float(ref[2]), 1, *w.dims, 0, V, prec, hp, stream)))
print("empty sync              %.3f ms" % t(lambda: None))
n = 300
for _ in range(20):
    ndf.reconstruct_field(model, ref, ndf.ROLE_MU, w.dims)
import time as _t
t0 = _t.perf_counter()
for _ in range(n):
    ndf.reconstruct_field(model, ref, ndf.ROLE_MU, w.dims)
print("reconstruct_field x%d mean %.4f ms" % (n, (_t.perf_counter() - t0) * 1e3 / n))
t0 = _t.perf_counter()
for _ in range(n):
    lib.ndf_query_grid(desc, float(ref[0]), float(ref[1]), float(ref[2]), 1, *w.dims, 0, V, prec, hp, stream)
    torch.cuda.current_stream().synchronize()
print("raw C-ABI x%d mean %.4f ms" % (n, (_t.perf_counter() - t0) * 1e3 / n))
