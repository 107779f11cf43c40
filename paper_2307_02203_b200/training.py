"""Training-target generation on the GPU: drop-ins for the reference's target path,
``training._targets`` (training.py:111-119) and ``sample_pairs_with_targets``
(training.py:122-150) -- the caller of the bulk estimators.

The reference samples both position sets with ``sample_many`` (fp64 trilinear over all
M members, ensemble.py:130-167) and then runs ``pearson_rowwise`` (measures.py:111-133)
or a Python loop of ``ksg_mi`` (measures.py:173-203), one pair at a time.  Here the
samples stay in HBM (``ndf_sample_many_vm`` writes the (B, M) fp64 rows from the variable's
vertex-major copy, built once for large batches; ``ndf_sample_many_ld`` otherwise) and ONE
``ndf_pearson_rows`` or ``ndf_ksg_rows`` launch per chunk evaluates every pair: Pearson
within 1e-12 of the reference (NaN for a constant row, exactly 1.0 for identical rows,
as ``pearson_rowwise``), KSG MI bit-identical.  ``sample_pairs_with_targets`` keeps the
reference's draws and resampling loop (same Generator calls in the same order), so a
caller gets the same positions for the same RNG state.  Training itself (Adam, backward
passes) stays out of scope.
"""

from __future__ import annotations

import logging

import numpy as np

from . import _native as N
from .ensemble import _device_view
from .errors import DataError, ParameterError
from .measures import CorrelationMeasure, _KsgTables

log = logging.getLogger(__name__)

_RESAMPLE_ROUNDS = 10            # training.py:28
DEFAULT_CHUNK = 65536            # pairs per launch: 2 x 65536 x M fp64 rows (1 GB at M = 1000)


def targets_device(field_obj, measure: CorrelationMeasure, var_mu: str, var_nu: str, p_mu, p_nu,
                   chunk: int = DEFAULT_CHUNK):
    """Targets of the position pairs (p_mu[i], p_nu[i]) as a CUDA fp64 tensor (B,)."""
    import torch
    p_mu = np.atleast_2d(np.asarray(p_mu, dtype=np.float64))
    p_nu = np.atleast_2d(np.asarray(p_nu, dtype=np.float64))
    if p_mu.shape != p_nu.shape or p_mu.shape[1] != 3:
        raise ParameterError(f"positions must be two (B, 3) arrays, got {p_mu.shape} and {p_nu.shape}")
    if measure.kind not in ("pearson", "ksg_mi"):
        raise ParameterError(f"unknown measure {measure.kind!r}")
    dmu, dnu = _device_view(field_obj, var_mu), _device_view(field_obj, var_nu)
    if dmu.member_count != dnu.member_count:
        raise ParameterError("variables differ in member count")
    dev = dmu.device
    M = dmu.member_count
    B = p_mu.shape[0]
    out = torch.empty(B, dtype=torch.float64, device=dev)
    if B == 0:
        return out
    stream = N.stream_handle(dev)
    # large batches: sample from a vertex-major copy (built once per variable, kept by the
    # DeviceEnsemble) -- every lattice corner's members are one contiguous row there
    for d_ in (dmu, dnu):
        if B * M >= d_.node_count and d_.col0 == 0 and d_.ld == d_.node_count:
            d_.vertex_major()
    if measure.kind == "ksg_mi":
        k = measure.ksg_k
        if not 1 <= k <= M - 1:
            raise ParameterError(f"need 1 <= k <= N-1, got k={k}, N={M}")
        jit, psi = _KsgTables.get(dev, M)
        psi_km = _KsgTables.psi_km(k, M)
        status = torch.zeros(1, dtype=torch.int32, device=dev)
    step = max(1, int(chunk))
    for s in range(0, B, step):
        e = min(B, s + step)
        a = dmu.sample_many(p_mu[s:e])               # (n, M) fp64, bit-identical samples
        b = dnu.sample_many(p_nu[s:e])
        n = e - s
        if measure.kind == "pearson":
            N.call("ndf_pearson_rows", N.ptr(a), M, N.ptr(b), M, n, N.ptr(out[s:e]), stream)
        else:
            N.call("ndf_ksg_rows", N.ptr(a), M, N.ptr(b), M, n, k, N.ptr(jit), N.ptr(psi), psi_km,
                   N.ptr(out[s:e]), None, None, N.ptr(status), stream)
    if measure.kind == "ksg_mi" and int(status.item()):
        raise ParameterError("digamma defined here for positive arguments only")
    return out


def targets(field_obj, measure: CorrelationMeasure, var_mu: str, var_nu: str, p_mu,
            p_nu) -> np.ndarray:
    """training.py:111-119 -- fp64 targets of the position pairs, on the host."""
    return targets_device(field_obj, measure, var_mu, var_nu, p_mu, p_nu).cpu().numpy()


def _uniform_pairs(rng: np.random.Generator, count: int):
    """training.py:90-92 (same Generator call)."""
    pts = rng.uniform(-1.0, 1.0, size=(count, 6))
    return pts[:, :3].copy(), pts[:, 3:].copy()


def _grid_pairs(rng: np.random.Generator, count: int, field_obj):
    """training.py:95-108: pairs on ensemble node coordinates (same Generator calls)."""
    dom = field_obj.domain
    out = []
    for _ in range(2):
        ix = rng.integers(0, dom.nx, count)
        iy = rng.integers(0, dom.ny, count)
        iz = rng.integers(0, dom.nz, count)
        out.append(np.column_stack([
            2.0 * ix / (dom.nx - 1) - 1.0,
            2.0 * iy / (dom.ny - 1) - 1.0,
            2.0 * iz / (dom.nz - 1) - 1.0,
        ]))
    return out[0], out[1]


def sample_pairs_with_targets(field_obj, config, rng: np.random.Generator, count: int,
                              on_grid: bool = False):
    """training.py:122-150: draw position pairs and their targets, resampling degenerate
    pairs; ``config`` supplies ``measure``, ``var_mu`` and ``var_nu`` (the reference's
    ``TrainingConfig`` works as is).  Raises DataError if degenerate targets persist."""
    draw = _grid_pairs if on_grid else _uniform_pairs
    args = (rng, count, field_obj) if on_grid else (rng, count)
    p_mu, p_nu = draw(*args)
    tg = targets(field_obj, config.measure, config.var_mu, config.var_nu, p_mu, p_nu)
    for _ in range(_RESAMPLE_ROUNDS):
        bad = ~np.isfinite(tg)
        if not bad.any():
            return p_mu, p_nu, tg
        n_bad = int(bad.sum())
        log.warning("resampling %d degenerate target pairs", n_bad)
        redraw_args = (rng, n_bad, field_obj) if on_grid else (rng, n_bad)
        p_mu[bad], p_nu[bad] = draw(*redraw_args)
        tg[bad] = targets(field_obj, config.measure, config.var_mu, config.var_nu, p_mu[bad],
                          p_nu[bad])
    if not np.isfinite(tg).all():
        raise DataError("degenerate targets persisted through resampling")
    return p_mu, p_nu, tg
