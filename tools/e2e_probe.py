import time, statistics, os, sys
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_2307_02203_b200 as ndf
from paper_2307_02203_b200 import workloads as W
w = W.CONFIGS[1]
m = W.build_model(w, seed=0, grid_init=1e-4).with_precision("bf16")
ref = w.ref_position()
flush = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
def tm(f, n=30):
    ts = []
    for i in range(n + 5):
        flush.fill_(float(i)); torch.cuda.synchronize()
        t0 = time.perf_counter(); f(); ts.append((time.perf_counter() - t0) * 1e3)
    return statistics.mean(ts[5:])
out = torch.empty(w.n_vertices, dtype=torch.float32, device="cuda")
pin = torch.empty(w.n_vertices, dtype=torch.float32, pin_memory=True)
def dev():
    ndf.reconstruct_field_device(m, ref, ndf.ROLE_MU, w.dims, out=out); torch.cuda.synchronize()
def pinned():
    ndf.reconstruct_field_device(m, ref, ndf.ROLE_MU, w.dims, out=pin); torch.cuda.synchronize()
def public():
    ndf.reconstruct_field(m, ref, ndf.ROLE_MU, w.dims)
def resp():
    ndf.reconstruct_response(m, ref, ndf.ROLE_MU, w.dims)
for name, f in [("device out + sync", dev), ("pinned out + sync", pinned), ("reconstruct_field", public), ("reconstruct_response", resp)]:
    print(f"{name:24s} {tm(f):.4f} ms")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ks = []
for i in range(30):
    flush.fill_(1.0); e0.record(); ndf.reconstruct_field_device(m, ref, ndf.ROLE_MU, w.dims, out=pin); e1.record(); torch.cuda.synchronize(); ks.append(e0.elapsed_time(e1))
print("pinned out, events", statistics.mean(ks[5:]))
ks = []
for i in range(30):
    flush.fill_(1.0); e0.record(); ndf.reconstruct_field_device(m, ref, ndf.ROLE_MU, w.dims, out=out); e1.record(); torch.cuda.synchronize(); ks.append(e0.elapsed_time(e1))
print("device out, events", statistics.mean(ks[5:]))
