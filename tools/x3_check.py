"""bf16 split-operand query (query_x3_kernel): parity vs the oracle and timing vs fp16.

    python tools/x3_check.py [n_oracle_vertices]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_02203_b200 as ndf  # noqa: E402
from oracle import ndf_oracle as O  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402


def om(model):
    return O.OracleModel(model.spec.fourier_octaves, model.grid_mu, model.grid_nu, model.weights,
                         model.biases, model.spec.merge, model.spec.activation,
                         model.spec.head_kind)


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


nver = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
w0 = W.CONFIGS[0]
m0 = W.build_model(w0, seed=0, grid_init=1.0)
want = O.reconstruct_field(om(m0), w0.ref_position(), w0.dims)
for prec in ("fp16", "bf16"):
    got = ndf.reconstruct_field(m0.with_precision(prec), w0.ref_position(), ndf.ROLE_MU, w0.dims).values
    print(f"c0 {prec}: max|err| vs oracle {np.abs(got - want).max():.3e}", flush=True)

for cfg in (1, 2):
    w = W.CONFIGS[cfg]
    idx = np.sort(np.random.default_rng(5).choice(w.n_vertices, nver, replace=False))
    for gi in (1.0, 1e-4):
        m = W.build_model(w, seed=0, grid_init=gi)
        t0 = time.time()
        want = O.reconstruct_field(om(m), w.ref_position(), w.dims, vertices=idx)
        tw = time.time() - t0
        for prec in ("fp16", "bf16"):
            mp = m.with_precision(prec)
            out = ndf.reconstruct_field_device(mp, w.ref_position(), ndf.ROLE_MU, w.dims)
            err = np.abs(out.cpu().numpy()[idx] - want).max()
            ms = timeit(lambda: ndf.reconstruct_field_device(mp, w.ref_position(), ndf.ROLE_MU,
                                                             w.dims, out=out))
            print(f"c{cfg} gi={gi:g} {prec}: max|err| vs oracle ({nver} vtx) {err:.3e}  "
                  f"{ms:.4f} ms/query  (oracle {tw:.1f}s)", flush=True)

# multi-reference cube rows == single queries (fp16-rounded)
w = W.CONFIGS[1]
dims = (64, 40, 6)
m = W.build_model(w, seed=0, grid_init=1.0).with_precision("bf16")
spec = ndf.ModelSpec.baseline(dims, 4, precision="bf16", grid_init=1.0)
m = ndf.NdfModel.build(spec, seed=3)
refs = O.grid_positions(dims)[[5, 777, 9000, 15359]]
cube = ndf.reconstruct_multi_device(m, refs, ndf.ROLE_MU, dims).cpu().numpy()
for k, r in enumerate(refs):
    one = ndf.reconstruct_field(m, r, ndf.ROLE_MU, dims).values.astype(np.float16)
    print(f"cube row {k}: equal to single query: {np.array_equal(cube[k], one)}", flush=True)
