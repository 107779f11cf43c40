"""Ensemble containers, NDFE IO and GPU-resident ensembles.

Mirrors the reference's ``ensemble.py`` (GridDomain ``:34-62``, EnsembleField
``:65-112``, NDFE ``save_ensemble``/``load_ensemble`` ``:283-333``,
``sample_many``/``sample_at`` ``:130-173``) with the same semantics, plus
``DeviceEnsemble``: one variable's member-major fp32 block resident in HBM
(the NDFE payload layout, ``(M, nz, ny, nx)``), with lazily built derived
layouts (standardised Z for the Pearson GEMV, vertex-major copy for pair lists).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .errors import (CorruptFileError, DataError, FormatError, ParameterError,
                     UnknownVariableError)

NDFE_MAGIC = b"NDFE"
NDFE_VERSION = 1


@dataclass(frozen=True)
class GridDomain:
    """Node counts of a regular grid over Omega = [-1, 1]^3 (ensemble.py:34-62)."""

    nx: int
    ny: int
    nz: int

    def __post_init__(self):
        for n in (self.nx, self.ny, self.nz):
            if int(n) != n or n < 2:
                raise ParameterError(f"grid axes need >= 2 nodes, got {self!r}")

    @property
    def node_count(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def dims(self):
        return (self.nx, self.ny, self.nz)

    def axis_coords(self, axis: int) -> np.ndarray:
        n = (self.nx, self.ny, self.nz)[axis]
        return 2.0 * np.arange(n) / (n - 1) - 1.0

    def node_positions(self) -> np.ndarray:
        zs, ys, xs = np.meshgrid(self.axis_coords(2), self.axis_coords(1),
                                 self.axis_coords(0), indexing="ij")
        return np.column_stack([xs.ravel(), ys.ravel(), zs.ravel()])


@dataclass(frozen=True)
class EnsembleField:
    """N member grids per variable, float32 (d, N, nz, ny, nx) (ensemble.py:65-112)."""

    domain: GridDomain
    variables: tuple
    values: np.ndarray = field(repr=False)

    def __post_init__(self):
        vals = np.asarray(self.values, dtype=np.float32)
        object.__setattr__(self, "values", vals)
        object.__setattr__(self, "variables", tuple(self.variables))
        if len(set(self.variables)) != len(self.variables):
            raise DataError(f"duplicate variable names: {self.variables}")
        if vals.ndim != 5:
            raise DataError(f"values must be (d, N, nz, ny, nx), got {vals.shape}")
        d, n, nz, ny, nx = vals.shape
        if d != len(self.variables):
            raise DataError(f"{len(self.variables)} variable names but {d} value blocks")
        if (nx, ny, nz) != (self.domain.nx, self.domain.ny, self.domain.nz):
            raise DataError(f"grid shape {(nx, ny, nz)} does not match domain {self.domain}")
        if n < 1:
            raise DataError("ensemble needs at least one member")
        if not np.isfinite(vals).all():
            raise DataError("ensemble contains non-finite values")
        object.__setattr__(self, "_device_cache", {})

    @property
    def member_count(self) -> int:
        return self.values.shape[1]

    def variable_index(self, name: str) -> int:
        try:
            return self.variables.index(name)
        except ValueError:
            raise UnknownVariableError(
                f"unknown variable {name!r}; have {list(self.variables)}") from None

    def member_grids(self, name: str) -> np.ndarray:
        return self.values[self.variable_index(name)]

    def to_device(self, variable: str, device=None) -> "DeviceEnsemble":
        """Upload one variable once (cached per device): the HBM-resident copy."""
        dev = N.require_cuda(device)
        key = (variable, str(dev))
        cache = self._device_cache
        if key not in cache:
            cache[key] = DeviceEnsemble.from_numpy(self.member_grids(variable), device=dev)
        return cache[key]


class DeviceEnsemble:
    """One variable's ensemble resident on a CUDA device, member-major fp32.

    ``X`` is a torch tensor of shape (M, nz, ny, nx) -- the NDFE payload layout,
    so member rows are contiguous over vertices (coalesced GEMV / KSG loads) -- or,
    for a V-slice of a sharded ensemble, (M, cols) holding node columns
    [col0, col0 + cols) of the same layout (``window``).
    """

    def __init__(self, X, domain: GridDomain, col0: int = 0):
        import torch
        if X.dtype != torch.float32 or not X.is_cuda:
            raise DataError("DeviceEnsemble needs a float32 CUDA tensor")
        if X.dim() == 4:
            M, nz, ny, nx = X.shape
            if (nx, ny, nz) != domain.dims or col0 != 0:
                raise DataError("tensor shape does not match domain")
        elif X.dim() != 2 or col0 < 0 or col0 + X.shape[1] > domain.node_count:
            raise DataError("column window must be (M, cols) inside the domain")
        self.X = X.contiguous()
        self.domain = domain
        self.col0 = int(col0)
        self.ld = int(X.shape[1]) if X.dim() == 2 else domain.node_count
        self._z = None
        self._norm = None
        self._xv = None

    @classmethod
    def window(cls, grids, c0: int, c1: int, device=None) -> "DeviceEnsemble":
        """Upload node columns [c0, c1) of host member grids (N, nz, ny, nx): the V-slice
        one rank of a sharded ensemble holds (0.88 GB per GPU for config 1 at 8 GPUs)."""
        import torch
        dev = N.require_cuda(device)
        g = np.asarray(grids)
        if g.ndim != 4:
            raise DataError("member grids must be (N, nz, ny, nx)")
        dom = GridDomain(g.shape[3], g.shape[2], g.shape[1])
        if not 0 <= c0 < c1 <= dom.node_count:
            raise ParameterError("column window out of range")
        cols = np.ascontiguousarray(g.reshape(g.shape[0], -1)[:, c0:c1], dtype=np.float32)
        return cls(torch.from_numpy(cols).to(dev), dom, c0)

    @property
    def full(self) -> bool:
        return self.col0 == 0 and self.ld == self.domain.node_count

    def _need_full(self, what):
        if not self.full:
            raise ParameterError(f"{what} needs the whole variable, not a column window")

    @classmethod
    def from_numpy(cls, grids: np.ndarray, device=None) -> "DeviceEnsemble":
        import torch
        dev = N.require_cuda(device)
        g = np.ascontiguousarray(grids, dtype=np.float32)
        if g.ndim != 4:
            raise DataError("member grids must be (N, nz, ny, nx)")
        t = torch.from_numpy(g).to(dev, non_blocking=False)
        return cls(t, GridDomain(g.shape[3], g.shape[2], g.shape[1]))

    @property
    def member_count(self) -> int:
        return int(self.X.shape[0])

    @property
    def node_count(self) -> int:
        return self.domain.node_count

    @property
    def device(self):
        return self.X.device

    def zscore(self):
        """(Z, norm): standardised copy for the Pearson GEMV, built once (ndf_zscore)."""
        import torch
        self._need_full("zscore")
        if self._z is None:
            M, V = self.member_count, self.node_count
            Z = torch.empty((M, V), dtype=torch.float32, device=self.device)
            norm = torch.empty((V,), dtype=torch.float32, device=self.device)
            N.call("ndf_zscore", N.ptr(self.X), M, V, 0, V, N.ptr(Z), N.ptr(norm),
                   N.stream_handle(self.device))
            self._z, self._norm = Z, norm
        return self._z, self._norm

    def vertex_major(self):
        """(V, M) copy for pair lists, built once (ndf_vertex_major)."""
        import torch
        self._need_full("vertex_major")
        if self._xv is None:
            M, V = self.member_count, self.node_count
            Xv = torch.empty((V, M), dtype=torch.float32, device=self.device)
            N.call("ndf_vertex_major", N.ptr(self.X), M, V, N.ptr(Xv), N.stream_handle(self.device))
            self._xv = Xv
        return self._xv

    def drop_derived(self):
        self._z = self._norm = self._xv = None

    def sample_many(self, positions) -> "torch.Tensor":
        """Trilinear fp64 samples (B, M) on device (ndf_sample_many)."""
        import torch
        pos = _as_device_positions(positions, self.device)
        B = int(pos.shape[0])
        out = torch.empty((B, self.member_count), dtype=torch.float64, device=self.device)
        d = self.domain
        if self._xv is not None:         # vertex-major copy built: whole-row corner reads
            N.call("ndf_sample_many_vm", N.ptr(self._xv), self.member_count, d.nx, d.ny, d.nz,
                   N.ptr(pos), B, N.ptr(out), N.stream_handle(self.device))
        else:
            N.call("ndf_sample_many_ld", N.ptr(self.X), self.member_count, self.ld, self.col0,
                   d.nx, d.ny, d.nz, N.ptr(pos), B, N.ptr(out), N.stream_handle(self.device))
        return out


def _as_device_positions(positions, device):
    import torch
    if isinstance(positions, torch.Tensor):
        pos = positions.to(device=device, dtype=torch.float64)
    else:
        pos = torch.from_numpy(np.ascontiguousarray(np.atleast_2d(
            np.asarray(positions, dtype=np.float64)))).to(device)
    if pos.dim() != 2 or pos.shape[1] != 3:
        raise ParameterError(f"positions must be (M, 3), got {tuple(pos.shape)}")
    return pos.contiguous()


_FOREIGN_ENSEMBLES = {}   # (id(field), variable, device) -> (weakref, DeviceEnsemble)


def _device_view(field_obj, variable: str, device=None) -> DeviceEnsemble:
    """HBM view of one variable: a DeviceEnsemble, a {name: DeviceEnsemble} dict, this
    package's EnsembleField (cached upload), or the reference's own
    ``ndf.ensemble.EnsembleField`` (ensemble.py:65-112; duck-typed on ``domain`` and
    ``member_grids``; immutable, so its upload is cached per object until it is freed)."""
    if isinstance(field_obj, DeviceEnsemble):
        return field_obj
    if isinstance(field_obj, dict):          # {name: DeviceEnsemble}
        try:
            return field_obj[variable]
        except KeyError:
            raise UnknownVariableError(f"unknown variable {variable!r}") from None
    if hasattr(field_obj, "to_device"):
        return field_obj.to_device(variable, device)
    if not (hasattr(field_obj, "member_grids") and hasattr(field_obj, "domain")):
        raise ParameterError(f"not an ensemble field: {type(field_obj).__name__}")
    import weakref
    dev = N.require_cuda(device)
    key = (id(field_obj), variable, str(dev))
    hit = _FOREIGN_ENSEMBLES.get(key)
    if hit is not None and hit[0]() is field_obj:
        return hit[1]
    try:
        grids = field_obj.member_grids(variable)
    except Exception as exc:                 # the reference raises its own UnknownVariableError
        raise UnknownVariableError(str(exc)) from None
    d = field_obj.domain
    if tuple(np.shape(grids))[1:] != (d.nz, d.ny, d.nx):
        raise DataError("member grids do not match the field's domain")
    if not np.isfinite(grids).all():
        raise DataError("ensemble contains non-finite values")
    view = DeviceEnsemble.from_numpy(grids, device=dev)
    try:
        weakref.finalize(field_obj, _FOREIGN_ENSEMBLES.pop, key, None)
        _FOREIGN_ENSEMBLES[key] = (weakref.ref(field_obj), view)
    except TypeError:
        pass
    return view


def sample_many(field_obj, variable: str, positions, chunk: int = 8192) -> np.ndarray:
    """ensemble.py:130-167 on the GPU (fp64 trilinear, bit-identical); returns (M, N) fp64."""
    dev = _device_view(field_obj, variable)
    pos = np.atleast_2d(np.asarray(positions, dtype=np.float64))
    if pos.ndim != 2 or pos.shape[1] != 3:
        raise ParameterError(f"positions must be (M, 3), got {pos.shape}")
    return dev.sample_many(pos).cpu().numpy()


def sample_at(field_obj, variable: str, position) -> np.ndarray:
    """ensemble.py:170-173."""
    return sample_many(field_obj, variable,
                       np.asarray(position, dtype=np.float64).reshape(1, 3))[0]


# ---------------------------------------------------------------------------
# NDFE container (ensemble.py:283-333), byte-compatible with the reference


def save_ensemble(field_obj: EnsembleField, path) -> None:
    dom = field_obj.domain
    with open(path, "wb") as fh:
        fh.write(NDFE_MAGIC)
        fh.write(struct.pack("<6I", NDFE_VERSION, dom.nx, dom.ny, dom.nz,
                             field_obj.member_count, len(field_obj.variables)))
        for name in field_obj.variables:
            raw = name.encode("utf-8")
            fh.write(struct.pack("<H", len(raw)))
            fh.write(raw)
        fh.write(np.ascontiguousarray(field_obj.values, dtype="<f4").tobytes())


def _read_ndfe_header(fh):
    """NDFE header (ensemble.py:283-294): magic, <6I version nx ny nz n d, then d
    length-prefixed UTF-8 variable names.  Returns (nx, ny, nz, n, names)."""
    magic = fh.read(4)
    if magic != NDFE_MAGIC:
        raise FormatError(f"bad magic {magic!r}, expected {NDFE_MAGIC!r}")
    head = fh.read(24)
    if len(head) != 24:
        raise CorruptFileError("truncated header")
    version, nx, ny, nz, n, d = struct.unpack("<6I", head)
    if version != NDFE_VERSION:
        raise FormatError(f"unsupported NDFE version {version}")
    names = []
    for _ in range(d):
        raw_len = fh.read(2)
        if len(raw_len) != 2:
            raise CorruptFileError("truncated variable table")
        (name_len,) = struct.unpack("<H", raw_len)
        raw = fh.read(name_len)
        if len(raw) != name_len:
            raise CorruptFileError("truncated variable name")
        names.append(raw.decode("utf-8"))
    return nx, ny, nz, n, names


def load_ensemble_device(path, variable: str, device=None, chunk_bytes: int = 256 << 20):
    """Stream ONE variable of an NDFE file straight into HBM.

    Instead of reading the whole payload into host memory (load_ensemble, like the
    reference's ensemble.py:320-333, holds every variable, twice at peak), the
    variable's byte range is read in ``chunk_bytes`` pieces into two pinned buffers
    that alternate with asynchronous H2D copies on a side stream, so disk / page
    cache reads overlap the PCIe transfers.  Same validation as load_ensemble
    (truncation -> CorruptFileError, non-finite values -> DataError).
    """
    import os
    import torch
    dev = N.require_cuda(device)
    with open(path, "rb") as fh:
        nx, ny, nz, n, names = _read_ndfe_header(fh)
        data_off = fh.tell()
        try:
            domain = GridDomain(nx, ny, nz)
        except ParameterError as exc:
            raise CorruptFileError(str(exc)) from exc
        if variable not in names:
            raise UnknownVariableError(f"unknown variable {variable!r}; have {names}")
        per_var = n * nz * ny * nx * 4
        size = os.fstat(fh.fileno()).st_size
        if size - data_off != len(names) * per_var:
            raise CorruptFileError(f"payload holds {(size - data_off) // 4} float32 values, "
                                   f"expected {len(names) * per_var // 4}")
        X = torch.empty((n, nz, ny, nx), dtype=torch.float32, device=dev)
        dst = X.view(-1).view(torch.uint8)
        chunk = max(1 << 20, min(int(chunk_bytes), per_var))
        bufs = [torch.empty(chunk, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        views = [memoryview(b.numpy()) for b in bufs]
        done = [None, None]
        stream = torch.cuda.Stream(dev)
        # X came from the caching allocator on the current stream: a block it recycled
        # may still be in use by work queued there, so the side stream waits for it
        stream.wait_stream(torch.cuda.current_stream(dev))
        fh.seek(data_off + names.index(variable) * per_var)
        pos, i = 0, 0
        while pos < per_var:
            cnt = min(chunk, per_var - pos)
            if done[i] is not None:
                done[i].synchronize()           # this pinned buffer's last copy finished
            got = fh.readinto(views[i][:cnt])
            if got != cnt:
                raise CorruptFileError("NDFE payload truncated")
            with torch.cuda.stream(stream):
                dst[pos:pos + cnt].copy_(bufs[i][:cnt], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
            done[i] = ev
            pos += cnt
            i ^= 1
        stream.synchronize()
    if not bool(torch.isfinite(X).all()):
        raise DataError("ensemble file contains non-finite values")
    return DeviceEnsemble(X, domain)


def load_ensemble(path) -> EnsembleField:
    with open(path, "rb") as fh:
        nx, ny, nz, n, names = _read_ndfe_header(fh)
        d = len(names)
        expected = d * n * nz * ny * nx
        payload = fh.read()
        if len(payload) != expected * 4:
            raise CorruptFileError(
                f"payload holds {len(payload) // 4} float32 values, expected {expected}")
    values = np.frombuffer(payload, dtype="<f4").reshape(d, n, nz, ny, nx)
    if not np.isfinite(values).all():
        raise DataError("ensemble file contains non-finite values")
    try:
        domain = GridDomain(nx, ny, nz)
    except ParameterError as exc:
        raise CorruptFileError(str(exc)) from exc
    # the reference copies the payload (ensemble.py:333); frombuffer is read-only
    # and EnsembleField is immutable, so the zero-copy view is safe here.
    return EnsembleField(domain, tuple(names), values)
