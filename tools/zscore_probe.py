"""ndf_zscore on config 1 (M = 1000, V = 1.76 M): event-timed, plus a fp64 check of Z on
seeded columns.  NDF_ZS_BPS overrides the blocks per SM (tuning only)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2307_02203_b200 import _native as N  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402

w = W.CONFIGS[1]
ens = W.generate_device(w)
M, V = ens.member_count, ens.node_count
Z = torch.empty((M, V), dtype=torch.float32, device="cuda")
norm = torch.empty((V,), dtype=torch.float32, device="cuda")
s = N.stream_handle(ens.device)
run = lambda: N.call("ndf_zscore", N.ptr(ens.X), M, V, 0, V, N.ptr(Z), N.ptr(norm), s)  # noqa: E731
for _ in range(2):
    run()
torch.cuda.synchronize()
ts = []
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[len(ts) // 2]
gbs = 2 * 4.0 * M * V / (ms * 1e-3) / 1e9
X = ens.X.reshape(M, V)
idx = torch.randperm(V, generator=torch.Generator().manual_seed(5))[:4096].to("cuda")
cols = X[:, idx].double()
c = cols - cols.mean(0)
nrm = c.norm(dim=0)
want = c / nrm
err = (Z[:, idx].double() - want).abs().max().item()
nerr = ((norm[idx].double() - nrm).abs() / nrm).max().item()
print(f"zscore bps={os.environ.get('NDF_ZS_BPS', 'default')}: {ms:.3f} ms  {gbs:.0f} GB/s  "
      f"max|dZ| {err:.2e}  max rel dnorm {nerr:.2e}")
