"""BASELINE.json workloads: seeded synthetic ensembles, models and query sets.

The paper's CSEns ensemble is not available (no network); seeded synthetic
ensembles with its shape stand in:

* members = shared smooth mean + FFT-filtered white noise with Gaussian
  covariance lengths (lx, ly, lz) cells (amplitude filter exp(-l^2 k^2 / 4)
  per axis), z-normalised per vertex across members;
* config 2 applies y = x + 0.5 x^2 + 0.2 sin(3x) to the standard-normal field.

Two generator backends: NumPy on the host (config 0 -- reproducible on any
machine, and what the CPU tests use) and torch on the GPU (configs 1-4, which
are 7 GB per variable).  Both are seeded; they draw different streams, so a
config has one canonical backend (recorded in DESIGN.md).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .ensemble import DeviceEnsemble, EnsembleField, GridDomain


@dataclass(frozen=True)
class Workload:
    name: str
    dims: tuple            # (nx, ny, nz)
    members: int
    lengths: tuple         # covariance lengths in cells (x, y, z)
    latent_factor: int
    precision: str
    measure: str           # model head: pearson -> tanh, ksg_mi -> softplus
    nonlinear: bool = False
    ksg_k: int = 8
    ref_vertex: tuple = None   # (ix, iy, iz)
    seed: int = 0

    @property
    def n_vertices(self) -> int:
        return self.dims[0] * self.dims[1] * self.dims[2]

    def ref_position(self):
        ix, iy, iz = self.ref_vertex
        return tuple(2.0 * i / (n - 1) - 1.0 for i, n in zip((ix, iy, iz), self.dims))

    def ref_flat(self) -> int:
        ix, iy, iz = self.ref_vertex
        return ix + self.dims[0] * (iy + self.dims[1] * iz)


BIG = (250, 352, 20)
CONFIGS = {
    0: Workload("c0_pearson_cpu", (32, 44, 4), 50, (4, 4, 1), 8, "fp32", "pearson",
                ref_vertex=(16, 22, 2), seed=2307),
    1: Workload("c1_pearson_full", BIG, 1000, (8, 8, 2), 4, "bf16", "pearson",
                ref_vertex=(125, 176, 10), seed=2308),
    2: Workload("c2_mi_full", BIG, 1000, (8, 8, 2), 4, "bf16", "ksg_mi", nonlinear=True,
                ref_vertex=(125, 176, 10), seed=2309),
    3: Workload("c3_multi_ref", BIG, 1000, (8, 8, 2), 4, "bf16", "pearson",
                ref_vertex=(125, 176, 10), seed=2310),
    4: Workload("c4_bulk_pairs", BIG, 1000, (8, 8, 2), 4, "bf16", "ksg_mi", nonlinear=True,
                ref_vertex=(125, 176, 10), seed=2311),
}


def smooth_mean(dims) -> np.ndarray:
    """Deterministic shared smooth mean on Omega, shape (nz, ny, nx)."""
    nx, ny, nz = dims
    x = 2.0 * np.arange(nx) / (nx - 1) - 1.0
    y = 2.0 * np.arange(ny) / (ny - 1) - 1.0
    z = 2.0 * np.arange(nz) / (nz - 1) - 1.0 if nz > 1 else np.zeros(1)
    zz, yy, xx = np.meshgrid(z, y, x, indexing="ij")
    return 0.5 * np.sin(np.pi * xx) * np.cos(0.5 * np.pi * yy) + 0.25 * zz


def _filter(dims, lengths, xp, device=None):
    nx, ny, nz = dims
    lx, ly, lz = lengths
    if xp is np:
        kz = 2 * np.pi * np.fft.fftfreq(nz)
        ky = 2 * np.pi * np.fft.fftfreq(ny)
        kx = 2 * np.pi * np.fft.rfftfreq(nx)
        return (np.exp(-(lz * kz[:, None, None]) ** 2 / 4) * np.exp(-(ly * ky[None, :, None]) ** 2 / 4)
                * np.exp(-(lx * kx[None, None, :]) ** 2 / 4))
    import torch
    kz = 2 * np.pi * torch.fft.fftfreq(nz, device=device, dtype=torch.float64)
    ky = 2 * np.pi * torch.fft.fftfreq(ny, device=device, dtype=torch.float64)
    kx = 2 * np.pi * torch.fft.rfftfreq(nx, device=device, dtype=torch.float64)
    f = (torch.exp(-(lz * kz[:, None, None]) ** 2 / 4) * torch.exp(-(ly * ky[None, :, None]) ** 2 / 4)
         * torch.exp(-(lx * kx[None, None, :]) ** 2 / 4))
    return f.to(torch.float32)


def _transform(x, xp):
    return x + 0.5 * x * x + 0.2 * xp.sin(3.0 * x)


def generate_host(w: Workload) -> EnsembleField:
    """NumPy backend (config 0 scale): returns a one-variable EnsembleField ('v')."""
    nx, ny, nz = w.dims
    rng = np.random.default_rng(w.seed)
    noise = rng.standard_normal((w.members, nz, ny, nx))
    spec = np.fft.rfftn(noise, axes=(1, 2, 3)) * _filter(w.dims, w.lengths, np)
    x = np.fft.irfftn(spec, s=(nz, ny, nx), axes=(1, 2, 3))
    x = (x - x.mean(axis=0)) / x.std(axis=0)
    if w.nonlinear:
        x = _transform(x, np)
    else:
        x = x + smooth_mean(w.dims)[None]
    return EnsembleField(GridDomain(nx, ny, nz), ("v",), x[None].astype(np.float32))


def generate_device(w: Workload, device=None, chunk: int = 40) -> DeviceEnsemble:
    """torch-on-GPU backend (configs 1-4): member-major (M, nz, ny, nx) float32 in HBM."""
    import torch
    from . import _native as N
    dev = N.require_cuda(device)
    nx, ny, nz = w.dims
    gen = torch.Generator(device=dev)
    gen.manual_seed(w.seed)
    X = torch.empty((w.members, nz, ny, nx), dtype=torch.float32, device=dev)
    filt = _filter(w.dims, w.lengths, torch, dev)
    for m0 in range(0, w.members, chunk):
        m1 = min(w.members, m0 + chunk)
        noise = torch.randn((m1 - m0, nz, ny, nx), generator=gen, device=dev, dtype=torch.float32)
        spec = torch.fft.rfftn(noise, dim=(1, 2, 3)) * filt
        X[m0:m1] = torch.fft.irfftn(spec, s=(nz, ny, nx), dim=(1, 2, 3))
        del noise, spec
    mean = X.mean(dim=0, dtype=torch.float64)
    var = torch.zeros_like(mean)
    for m0 in range(0, w.members, chunk):
        m1 = min(w.members, m0 + chunk)
        var += ((X[m0:m1].double() - mean) ** 2).sum(0)
    inv = torch.rsqrt(var / w.members)
    mu = None if w.nonlinear else torch.from_numpy(smooth_mean(w.dims)).to(dev)
    for m0 in range(0, w.members, chunk):
        m1 = min(w.members, m0 + chunk)
        x = (X[m0:m1].double() - mean) * inv
        x = _transform(x, torch) if w.nonlinear else x + mu
        X[m0:m1] = x.to(torch.float32)
    return DeviceEnsemble(X, GridDomain(nx, ny, nz))


def build_model(w: Workload, seed: int = 0, grid_init: float = 1.0):
    """Seeded BASELINE model for a workload (weights seed 0)."""
    from .model import ModelSpec, NdfModel
    spec = ModelSpec.baseline(w.dims, w.latent_factor, measure_kind=w.measure,
                              precision=w.precision, grid_init=grid_init)
    return NdfModel.build(spec, seed=seed)


def reference_vertices(w: Workload, count: int = 64, seed: int = 1) -> np.ndarray:
    """Seeded-uniform reference vertices (config 3); flat indices."""
    return np.random.default_rng(seed).integers(0, w.n_vertices, size=count)


def pair_list(w: Workload, count: int = 1 << 22, seed: int = 2):
    """Config 4: half uniform pairs, half within +-16 cells per axis (clipped)."""
    rng = np.random.default_rng(seed)
    nx, ny, nz = w.dims
    V = w.n_vertices
    h = count // 2
    a_u = rng.integers(0, V, size=h)
    b_u = rng.integers(0, V, size=h)
    a_n = rng.integers(0, V, size=count - h)
    ax, ay, az = a_n % nx, (a_n // nx) % ny, a_n // (nx * ny)
    off = rng.integers(-16, 17, size=(count - h, 3))
    bx = np.clip(ax + off[:, 0], 0, nx - 1)
    by = np.clip(ay + off[:, 1], 0, ny - 1)
    bz = np.clip(az + off[:, 2], 0, nz - 1)
    b_n = bx + nx * (by + ny * bz)
    return np.concatenate([a_u, a_n]).astype(np.int64), np.concatenate([b_u, b_n]).astype(np.int64)
