"""ndf_pearson_pairs over config 4's 2^22-pair list on the vertex-major copy (event-timed)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2307_02203_b200 import _native as N  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
w = W.CONFIGS[4]
ens = W.generate_device(w)
Xv = ens.vertex_major()
M, V = ens.member_count, ens.node_count
pa, pb = W.pair_list(w, count=n, seed=2)
tpa, tpb = torch.from_numpy(pa).cuda(), torch.from_numpy(pb).cuda()
out = torch.empty(n, dtype=torch.float64, device="cuda")
s = N.stream_handle(ens.device)
run = lambda: N.call("ndf_pearson_pairs", N.ptr(Xv), M, V, N.ptr(tpa), N.ptr(tpb), n, N.ptr(out), s)  # noqa
run()
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[2]
algo = n * (2 * 4.0 * M + 16 + 8)
print(f"pearson_pairs {n} pairs: {ms:.3f} ms  {algo / ms / 1e6:.0f} GB/s algorithmic "
      f"({2 * 4 * M} B of rows per pair)")
