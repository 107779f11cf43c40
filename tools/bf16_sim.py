"""NumPy simulation of 16-bit operand rounding in the NDF decoder (config 0 model).

Rounds weights and/or activations to bf16 or fp16 (as the tcgen05 kind::f16 path does),
keeps fp32/fp64 accumulation, and reports max |error| vs the fp32 oracle.  Used to show
that the bf16 path's error (~1.2e-2) is operand quantisation, not a kernel defect.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ndf_oracle as O  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402


def rnd(x, dt):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(dt).float().numpy()


w = W.CONFIGS[0]
act = sys.argv[1] if len(sys.argv) > 1 else "silu"     # hidden activation to simulate
for gi in (1.0, 1e-4):
    m = W.build_model(w, seed=0, grid_init=gi)
    ref = w.ref_position()
    pos = O.grid_positions(w.dims)
    a = O.embed(np.asarray(ref).reshape(1, 3), m.grid_mu, 6)
    q = O.embed(pos, m.grid_nu, 6)
    x = O.merge("sum_absdiff", np.broadcast_to(a, q.shape), q)
    exact = O.head("tanh", O.mlp_forward(m.weights, m.biases, act, x))[:, 0]

    def sim(round_w, round_a, dt):
        h = rnd(x, dt) if round_a else x
        L = len(m.weights)
        for i, (wt, b) in enumerate(zip(m.weights, m.biases)):
            ww = rnd(wt, dt) if (round_w and i < L - 1) else wt
            z = (h.astype(np.float64) @ ww.astype(np.float64) + b).astype(np.float32)
            if i == L - 1:
                return np.tanh(z)[:, 0]
            h = O.activation(act, z)
            if round_a and i < L - 2:
                h = rnd(h, dt)

    for name, args in [("weights only", (1, 0)), ("activations only", (0, 1)), ("both", (1, 1))]:
        print(f"grid_init={gi:g} {name:17s} bf16 {np.abs(sim(*args, torch.bfloat16) - exact).max():.3e}"
              f"  fp16 {np.abs(sim(*args, torch.float16) - exact).max():.3e}")
