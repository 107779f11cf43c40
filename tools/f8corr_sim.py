"""NumPy/torch simulation of the hidden-layer operand schemes of the bf16 grid query.

Compares, on a seeded vertex subset of a config's grid, max |error| vs the fp32 oracle for
  plain  : bf16(A) bf16(W)
  x3     : A_hi W_hi + A_lo W_hi + A_hi W_lo   (the shipped split kernel, all bf16)
  f8e5   : bf16(A) bf16(W) + [e5m2(A_lo) | e5m2(A_hi)] . [e5m2(W_hi) ; e5m2(W_lo)]
  f8e4s  : same with e4m3 and a power-of-two scale 2^s on A_lo / W_lo (D scaled by 2^s)
Layer 0 is exact (the kernel's selector + split latent MMAs), the output layer an fp32 dot.
Usage: python tools/f8corr_sim.py [config] [n_vertices]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ndf_oracle as O  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402

T = torch.float64


def q(x, dt, sat=None):
    x = torch.as_tensor(x, dtype=torch.float32)
    if sat is not None:
        x = x.clamp(-sat, sat)
    return x.to(dt).to(T)


def hidden(h, w, b, scheme, s=8):
    h32 = torch.as_tensor(h, dtype=torch.float32)
    w32 = torch.as_tensor(w, dtype=torch.float32)
    ah = q(h32, torch.bfloat16)
    wh = q(w32, torch.bfloat16)
    al = (h32.to(T) - ah).float()
    wl = (w32.to(T) - wh).float()
    b = torch.as_tensor(b, dtype=T)
    if scheme == "plain":
        z = ah @ wh
    elif scheme == "x3":
        z = ah @ wh + q(al, torch.bfloat16) @ wh + ah @ q(wl, torch.bfloat16)
    elif scheme == "f8e5":
        f = torch.float8_e5m2
        z = ah @ wh + q(al, f, 57344.) @ q(w32, f, 57344.) + q(h32, f, 57344.) @ q(wl, f, 57344.)
    elif scheme == "f8e4s":
        f = torch.float8_e4m3fn
        sc = float(2 ** s)
        z = ah @ wh + (q(al * sc, f, 448.) @ q(w32, f, 448.) + q(h32, f, 448.) @ q(wl * sc, f, 448.)) / sc
    else:
        raise ValueError(scheme)
    return (z + b).float().numpy()


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    nv = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 16
    w = W.CONFIGS[cfg]
    rng = np.random.default_rng(5)
    verts = np.sort(rng.choice(w.n_vertices, size=min(nv, w.n_vertices), replace=False))
    pos = O.grid_positions_of(w.dims, verts)
    for gi in (1.0, 1e-4):
        m = W.build_model(w, seed=0, grid_init=gi)
        act, headk = m.spec.activation, m.spec.head_kind
        a = O.embed(np.asarray(w.ref_position()).reshape(1, 3), m.grid_mu, m.spec.fourier_octaves)
        qe = O.embed(pos, m.grid_nu, m.spec.fourier_octaves)
        x = O.merge("sum_absdiff", np.broadcast_to(a, qe.shape), qe)
        exact = O.head(headk, O.mlp_forward(m.weights, m.biases, act, x))[:, 0]
        L = len(m.weights)
        res = {}
        for scheme in ("plain", "x3", "f8e5", "f8e4s"):
            z = (x.astype(np.float64) @ m.weights[0].astype(np.float64) + m.biases[0]).astype(np.float32)
            h = O.activation(act, z)
            for i in range(1, L - 1):
                h = O.activation(act, hidden(h, m.weights[i], m.biases[i], scheme))
            out = (h.astype(np.float64) @ m.weights[-1].astype(np.float64) + m.biases[-1]).astype(np.float32)
            res[scheme] = float(np.abs(O.head(headk, out)[:, 0] - exact).max())
        print(f"c{cfg} grid_init={gi:g} head={headk} n={len(verts)}: " +
              "  ".join(f"{k} {v:.2e}" for k, v in res.items()), flush=True)


if __name__ == "__main__":
    main()
