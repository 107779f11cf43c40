"""Ground-truth dependence estimators on the GPU (drop-in for measures.py).

Same names, argument meaning and error behaviour as the reference
(``pkg/src/ndf/measures.py``): ``pearson`` (:59-81), ``pearson_against``
(:84-108), ``pearson_rowwise`` (:111-133), ``digamma`` (:136-165), ``ksg_mi``
(:173-203), ``gaussian_mi_analytic`` (:206-210), ``FieldGrid`` (:216-237),
``grid_positions`` (:240-252), ``ground_truth_field`` (:273-315), NDFG IO
(:318-343).  Every estimate is computed by libndf_b200 kernels; the host only
validates arguments, builds constant tables (digamma values, the fixed
tie-breaking jitter) and moves results.
"""

from __future__ import annotations

import logging
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .ensemble import DeviceEnsemble, EnsembleField, _device_view
from .errors import (CorruptFileError, DegenerateSampleError, FormatError,
                     ParameterError, ShapeError)

log = logging.getLogger(__name__)

NDFG_MAGIC = b"NDFG"
NDFG_VERSION = 1
_JITTER_SEED = 0x5D17E3     # measures.py:33


@dataclass(frozen=True)
class CorrelationMeasure:
    """Estimator selection: Pearson's r or KSG mutual information (measures.py:36-56)."""

    kind: str = "pearson"
    ksg_k: int = 3

    def __post_init__(self):
        if self.kind not in ("pearson", "ksg_mi"):
            raise ParameterError(f"unknown measure kind {self.kind!r}")
        if self.ksg_k < 1:
            raise ParameterError("ksg_k must be >= 1")

    def __call__(self, a, b) -> float:
        if self.kind == "pearson":
            return pearson(a, b)
        return ksg_mi(a, b, self.ksg_k)

    @property
    def symmetric(self) -> bool:
        return True


# ---------------------------------------------------------------------------
# host-side constant tables


def digamma(x):
    """Digamma via recurrence + asymptotic series (measures.py:136-165), host fp64.

    Used to build the psi table the KSG kernel indexes; same formula and
    operation order as the reference, so table values are the reference's bits.
    """
    x = np.asarray(x, dtype=np.float64)
    if np.any(x <= 0.0):
        raise ParameterError("digamma defined here for positive arguments only")
    scalar = x.ndim == 0
    x = np.atleast_1d(x).copy()
    acc = np.zeros_like(x)
    for _ in range(10):
        small = x < 10.0
        if not small.any():
            break
        acc[small] -= 1.0 / x[small]
        x[small] += 1.0
    inv2 = 1.0 / (x * x)
    series = (np.log(x) - 0.5 / x
              - inv2 * (1.0 / 12.0 - inv2 * (1.0 / 120.0 - inv2 * (
                  1.0 / 252.0 - inv2 * (1.0 / 240.0 - inv2 / 132.0)))))
    out = acc + series
    return float(out[0]) if scalar else out


class _KsgTables:
    """Per-(device, M) constants: jitter r (measures.py:168-170) and psi(n+1)."""

    _cache: dict = {}

    @classmethod
    def get(cls, device, M: int):
        import torch
        key = (str(device), M)
        if key not in cls._cache:
            r = np.random.default_rng(_JITTER_SEED).random(M) - 0.5
            psi = digamma(np.arange(1, M + 1, dtype=np.float64))
            cls._cache[key] = (torch.from_numpy(r).to(device), torch.from_numpy(psi).to(device))
        return cls._cache[key]

    @staticmethod
    def psi_km(k: int, M: int) -> float:
        return digamma(float(k)) + digamma(float(M))


# ---------------------------------------------------------------------------
# scalar / row estimators


def _to_dev_f64(x, device):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(device)


def pearson(a, b) -> float:
    """measures.py:59-81."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    if a.shape != b.shape:
        raise ParameterError(f"length mismatch: {a.size} vs {b.size}")
    if a.size < 2:
        raise ParameterError("need at least two samples")
    r = pearson_rowwise(a[None, :], b[None, :])[0]
    if np.isnan(r):
        raise DegenerateSampleError("constant sample vector has no correlation")
    return float(r)


def pearson_against(ref, samples) -> np.ndarray:
    """measures.py:84-108: r of ref against each row; NaN for degenerate rows."""
    import torch
    ref = np.asarray(ref, dtype=np.float64).ravel()
    samples = np.atleast_2d(np.asarray(samples, dtype=np.float64))
    if samples.shape[1] != ref.size:
        raise ParameterError(f"length mismatch: {ref.size} vs {samples.shape[1]}")
    dev = N.require_cuda()
    B, M = samples.shape
    out = torch.empty(B, dtype=torch.float64, device=dev)
    if B:
        # keep the device copies referenced until the kernel is enqueued
        dref, dsmp = _to_dev_f64(ref, dev), _to_dev_f64(samples, dev)
        N.call("ndf_pearson_rows", N.ptr(dref), 0, N.ptr(dsmp), M, B, N.ptr(out),
               N.stream_handle(dev))
    return out.cpu().numpy()


def pearson_rowwise(a, b) -> np.ndarray:
    """measures.py:111-133."""
    import torch
    a = np.atleast_2d(np.asarray(a, dtype=np.float64))
    b = np.atleast_2d(np.asarray(b, dtype=np.float64))
    if a.shape != b.shape:
        raise ParameterError(f"shape mismatch: {a.shape} vs {b.shape}")
    dev = N.require_cuda()
    B, M = a.shape
    out = torch.empty(B, dtype=torch.float64, device=dev)
    if B:
        da, db = _to_dev_f64(a, dev), _to_dev_f64(b, dev)
        N.call("ndf_pearson_rows", N.ptr(da), M, N.ptr(db), M, B, N.ptr(out), N.stream_handle(dev))
    return out.cpu().numpy()


def ksg_mi(a, b, k: int = 3) -> float:
    """KSG mutual information (variant 1) in nats -- measures.py:173-203."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    if a.shape != b.shape:
        raise ParameterError(f"length mismatch: {a.size} vs {b.size}")
    n = a.size
    if not 1 <= k <= n - 1:
        raise ParameterError(f"need 1 <= k <= N-1, got k={k}, N={n}")
    mi, _ = ksg_rows(a[None, :], b[None, :], k)
    return float(mi[0])


def ksg_rows(a, b, k: int, return_counts: bool = False):
    """Row-batched ksg_mi: a is (B, M) or (M,) (broadcast), b is (B, M).

    Returns (mi fp64 (B,), counts (B, 2, M) int32 or None).  Raises
    ParameterError where the reference's digamma would (a count of -1).
    """
    import torch
    b = np.atleast_2d(np.asarray(b, dtype=np.float64))
    a = np.asarray(a, dtype=np.float64)
    B, M = b.shape
    if not 1 <= k <= M - 1:
        raise ParameterError(f"need 1 <= k <= N-1, got k={k}, N={M}")
    dev = N.require_cuda()
    a_stride = 0 if a.ndim == 1 else M
    if a.ndim == 2 and a.shape != b.shape:
        raise ParameterError(f"shape mismatch: {a.shape} vs {b.shape}")
    jit, psi = _KsgTables.get(dev, M)
    mi = torch.empty(B, dtype=torch.float64, device=dev)
    counts = torch.empty((B, 2, M), dtype=torch.int32, device=dev) if return_counts else None
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    da, db = _to_dev_f64(a, dev), _to_dev_f64(b, dev)
    N.call("ndf_ksg_rows", N.ptr(da), a_stride, N.ptr(db), M, B, k,
           N.ptr(jit), N.ptr(psi), _KsgTables.psi_km(k, M), N.ptr(mi), None, N.ptr(counts),
           N.ptr(status), N.stream_handle(dev))
    if int(status.item()):
        raise ParameterError("digamma defined here for positive arguments only")
    return mi.cpu().numpy(), (counts.cpu().numpy() if counts is not None else None)


def gaussian_mi_analytic(rho: float) -> float:
    """measures.py:206-210."""
    if not abs(rho) < 1.0:
        raise ParameterError(f"|rho| must be < 1, got {rho}")
    return -0.5 * np.log1p(-rho * rho)


# ---------------------------------------------------------------------------
# dense field grids


@dataclass(frozen=True)
class FieldGrid:
    """Dense X*Y*Z scalar volume, values flat in x-fastest order (measures.py:216-237)."""

    dims: tuple
    values: np.ndarray = field(repr=False)

    def __post_init__(self):
        dims = tuple(int(d) for d in self.dims)
        object.__setattr__(self, "dims", dims)
        if any(d < 1 for d in dims):
            raise ParameterError(f"grid dims must be >= 1, got {dims}")
        vals = np.asarray(self.values, dtype=np.float32).ravel()
        if vals.size != dims[0] * dims[1] * dims[2]:
            raise ParameterError(f"expected {dims[0] * dims[1] * dims[2]} values, got {vals.size}")
        object.__setattr__(self, "values", vals)

    def as_zyx(self) -> np.ndarray:
        x, y, z = self.dims
        return self.values.reshape(z, y, x)


def grid_positions(dims) -> np.ndarray:
    """measures.py:240-252 (host; the query kernels recompute nodes on device)."""
    def axis(n):
        if n == 1:
            return np.zeros(1)
        return 2.0 * np.arange(n) / (n - 1) - 1.0

    x, y, z = dims
    zz, yy, xx = np.meshgrid(axis(z), axis(y), axis(x), indexing="ij")
    return np.column_stack([xx.ravel(), yy.ravel(), zz.ravel()])


def _check_dims(dims):
    dims = tuple(int(d) for d in dims)
    if len(dims) != 3 or any(d < 1 for d in dims):
        raise ParameterError(f"grid dims must be >= 1, got {dims}")
    return dims


def ground_truth_field_device(field_obj, measure: CorrelationMeasure, var_mu: str, var_nu: str,
                              ref, dims, v0: int = 0, v1: int | None = None,
                              chunk: int = 65536, ref_vec=None):
    """Device-resident ground truth for vertices [v0, v1) of ``dims`` (float32 CUDA tensor).

    Node-aligned grids (dims == the ensemble domain) read the ensemble
    directly: Pearson in one streaming pass over the member columns
    (ndf_pearson_field), KSG through the per-node kernel.  Other grids sample
    trilinearly first (bit-identical to sample_many) and run the row kernels on
    the samples.  Degenerate Pearson entries are NaN here; ``ground_truth_field``
    maps them to 0 with a warning.  ``field_obj`` may be a column window
    (DeviceEnsemble.window) covering [v0, v1); ``ref_vec`` (fp64 CUDA, M) then
    supplies the reference's member vector, e.g. broadcast from the rank holding it.
    """
    import torch
    dims = _check_dims(dims)
    V = dims[0] * dims[1] * dims[2]
    v1 = V if v1 is None else v1
    ref = np.asarray(ref, dtype=np.float64).reshape(3)
    dmu = _device_view(field_obj, var_mu)
    dnu = _device_view(field_obj, var_nu)
    dev = dnu.device
    stream = N.stream_handle(dev)
    M = dnu.member_count
    if ref_vec is None:
        ref_vec = dmu.sample_many(ref.reshape(1, 3))[0].contiguous()  # fp64 (M,)
    else:
        ref_vec = ref_vec.to(device=dev, dtype=torch.float64).contiguous()
        if ref_vec.shape != (M,):
            raise ShapeError(f"ref_vec must have {M} members, got {tuple(ref_vec.shape)}")
    out = torch.empty(v1 - v0, dtype=torch.float32, device=dev)
    node_aligned = dims == dnu.domain.dims
    if not node_aligned and not dnu.full:
        raise ParameterError("a column window serves node-aligned fields only")
    if node_aligned and v0 < v1 and not dnu.col0 <= v0 <= v1 <= dnu.col0 + dnu.ld:
        raise ParameterError("vertex range outside the ensemble's column window")
    if measure.kind == "pearson":
        if node_aligned:
            # one streaming read of the member columns, reference statistics on device
            # (ndf_pearson_field); no standardised copy, no host round trip
            N.call("ndf_pearson_field", N.ptr(dnu.X), M, dnu.ld, dnu.col0, N.ptr(ref_vec), v0, v1,
                   N.ptr(out), stream)
        else:
            pos = grid_positions(dims)[v0:v1]
            _vertex_major_for(dnu, len(pos))
            buf = torch.empty(min(chunk, max(len(pos), 1)), dtype=torch.float64, device=dev)
            for s in range(0, len(pos), chunk):
                rows = dnu.sample_many(pos[s:s + chunk])
                n = rows.shape[0]
                N.call("ndf_pearson_rows", N.ptr(ref_vec), 0, N.ptr(rows), M, n, N.ptr(buf), stream)
                out[s:s + n] = buf[:n].to(torch.float32)
    else:
        k = measure.ksg_k
        if k > M - 1:
            raise ParameterError(f"ksg_k={k} needs at least {k + 1} members, have {M}")
        jit, psi = _KsgTables.get(dev, M)
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        psi_km = _KsgTables.psi_km(k, M)
        if node_aligned:
            # columns of a window are addressed relative to its first column
            N.call("ndf_ksg_ref_nodes", N.ptr(dnu.X), M, dnu.ld, N.ptr(ref_vec), v0 - dnu.col0,
                   v1 - dnu.col0, k, N.ptr(jit), N.ptr(psi), psi_km, None, N.ptr(out), None,
                   N.ptr(status), stream)
        else:
            pos = grid_positions(dims)[v0:v1]
            _vertex_major_for(dnu, len(pos))
            for s in range(0, len(pos), chunk):
                rows = dnu.sample_many(pos[s:s + chunk])
                n = rows.shape[0]
                N.call("ndf_ksg_rows", N.ptr(ref_vec), 0, N.ptr(rows), M, n, k, N.ptr(jit), N.ptr(psi),
                       psi_km, None, N.ptr(out[s:s + n]), None, N.ptr(status), stream)
        if int(status.item()):
            raise ParameterError("digamma defined here for positive arguments only")
    return out


def _vertex_major_for(d, n_positions: int) -> None:
    """Off-node sampling of many positions reads whole member rows from the variable's
    vertex-major copy (ndf_sample_many_vm, bit-identical): build it once when the sampling
    would touch at least as many values as the copy costs to write."""
    if n_positions * d.member_count >= d.node_count and d.col0 == 0 and d.ld == d.node_count:
        d.vertex_major()


def ground_truth_field(field_obj, measure: CorrelationMeasure, var_mu: str, var_nu: str, ref,
                       dims, workers: int = 1, chunk: int = 4096) -> FieldGrid:
    """measures.py:273-315 on the GPU.

    ``workers`` / ``chunk`` are accepted for signature compatibility; results
    do not depend on them (as in the reference, measures.py:280-281).
    """
    dims = _check_dims(dims)
    out = ground_truth_field_device(field_obj, measure, var_mu, var_nu, ref, dims)
    vals = out.cpu().numpy()
    if measure.kind == "pearson":
        bad = np.isnan(vals)
        if bad.any():
            log.warning("ground truth: %d degenerate Pearson entries set to 0", int(bad.sum()))
            vals[bad] = 0.0
    return FieldGrid(dims, vals)


def save_field_grid(grid: FieldGrid, path) -> None:
    """measures.py:318-324."""
    x, y, z = grid.dims
    with open(path, "wb") as fh:
        fh.write(NDFG_MAGIC)
        fh.write(struct.pack("<4I", NDFG_VERSION, x, y, z))
        fh.write(np.ascontiguousarray(grid.values, dtype="<f4").tobytes())


def load_field_grid(path) -> FieldGrid:
    """measures.py:327-343."""
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != NDFG_MAGIC:
            raise FormatError(f"bad magic {magic!r}, expected {NDFG_MAGIC!r}")
        head = fh.read(16)
        if len(head) != 16:
            raise CorruptFileError("truncated NDFG header")
        version, x, y, z = struct.unpack("<4I", head)
        if version != NDFG_VERSION:
            raise FormatError(f"unsupported NDFG version {version}")
        payload = fh.read()
    if len(payload) != x * y * z * 4:
        raise CorruptFileError(f"payload holds {len(payload) // 4} values, expected {x * y * z}")
    return FieldGrid((x, y, z), np.frombuffer(payload, dtype="<f4").copy())


def pair_estimators_device(field_obj, variable: str, pa, pb, k: int = 8,
                           measures=("pearson", "ksg_mi"), counts: bool = False):
    """Bulk estimator pairs (BASELINE config 4 / training-target generation).

    For vertex pairs (pa[p], pb[p]) of one variable's node grid computes Pearson r
    (fp64, measures.py:111-133) and/or KSG MI (fp64, measures.py:173-203) on the
    GPU from a vertex-major copy of the ensemble.  Replaces the per-pair loop of
    training._targets (training.py:111-119).  Returns {name: CUDA fp64 tensor};
    ``counts=True`` adds "ksg_counts", the (n, 2, M) int32 KSG marginal counts n_x / n_y
    (measures.py:198-201) the MI was computed from.
    """
    import torch
    dev_ens = _device_view(field_obj, variable)
    dev = dev_ens.device
    V, M = dev_ens.node_count, dev_ens.member_count
    ta = torch.as_tensor(np.ascontiguousarray(pa, dtype=np.int64)).to(dev)
    tb = torch.as_tensor(np.ascontiguousarray(pb, dtype=np.int64)).to(dev)
    if ta.shape != tb.shape or ta.dim() != 1:
        raise ParameterError("pair index arrays must be equal-length vectors")
    if ta.numel() and (int(torch.minimum(ta.min(), tb.min())) < 0
                       or int(torch.maximum(ta.max(), tb.max())) >= V):
        raise ParameterError("pair index out of range")
    n = int(ta.numel())
    Xv = dev_ens.vertex_major()
    stream = N.stream_handle(dev)
    out = {}
    if "pearson" in measures:
        r = torch.empty(n, dtype=torch.float64, device=dev)
        N.call("ndf_pearson_pairs", N.ptr(Xv), M, V, N.ptr(ta), N.ptr(tb), n, N.ptr(r), stream)
        out["pearson"] = r
    if "ksg_mi" in measures:
        if not 1 <= k <= M - 1:
            raise ParameterError(f"need 1 <= k <= N-1, got k={k}, N={M}")
        jit, psi = _KsgTables.get(dev, M)
        mi = torch.empty(n, dtype=torch.float64, device=dev)
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        cnt = torch.empty((n, 2, M), dtype=torch.int32, device=dev) if counts else None
        N.call("ndf_ksg_pairs", N.ptr(Xv), M, V, N.ptr(ta), N.ptr(tb), n, k, N.ptr(jit),
               N.ptr(psi), _KsgTables.psi_km(k, M), N.ptr(mi), None, N.ptr(cnt), N.ptr(status),
               stream)
        if counts:
            out["ksg_counts"] = cnt
        if int(status.item()):
            raise ParameterError("digamma defined here for positive arguments only")
        out["ksg_mi"] = mi
    return out
