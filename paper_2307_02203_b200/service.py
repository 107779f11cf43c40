"""Reference-to-all-vertices reconstruction (drop-in for service.py's query path).

``reconstruct_field`` (service.py:46-84), ``difference_field`` (:87-94),
``matrix_reconstruct`` (:97-125) and ``benchmark`` (:186-220) with the
reference's signatures, plus the binary data plane of ``/api/reconstruct`` and
``/api/diff`` (:392-416) without the HTTP layer: ``reconstruct_response`` /
``difference_response``.  The query runs as ONE kernel launch over the whole
output grid: the reference point is embedded once per CTA, every query vertex
once, and the decoder runs fused on the tensor cores (fp16 / bf16 models) or in
exact fp32 (fp32 models).  ``batch_size`` is accepted for signature compatibility;
per-row arithmetic never depends on batching, so results are identical for any
value -- the property the reference guarantees (service.py:52-54).
"""

from __future__ import annotations

import statistics
import time
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import NotFoundError, ParameterError
from .measures import CorrelationMeasure, FieldGrid, ground_truth_field
from .model import NdfModel, as_model, ctypes_ref

DEFAULT_QUERY_BATCH = 65536
ROLE_MU = "reference-is-mu"
ROLE_NU = "reference-is-nu"


def _check_role(role: str) -> str:
    if role not in (ROLE_MU, ROLE_NU):
        raise ParameterError(f"role must be {ROLE_MU!r} or {ROLE_NU!r}")
    return role


def _check_dims(dims):
    dims = tuple(int(d) for d in dims)
    if len(dims) != 3 or any(d < 1 for d in dims):
        raise ParameterError(f"grid dims must be >= 1, got {dims}")
    return dims


def reconstruct_field_device(model: NdfModel, ref, role: str = ROLE_MU, dims=(64, 64, 64),
                             v0: int = 0, v1: int | None = None, out=None, clamp: bool = False):
    """Device-resident query of vertices [v0, v1) of ``dims``: float32 CUDA tensor.

    ``out`` (optional) is a preallocated float32 tensor of v1 - v0 values: CUDA, or
    pinned host memory (the kernel then writes host RAM directly; sync before reading).
    """
    import torch
    _check_role(role)
    model = as_model(model)
    dims = _check_dims(dims)
    V = dims[0] * dims[1] * dims[2]
    v1 = V if v1 is None else int(v1)
    if not 0 <= v0 <= v1 <= V:
        raise ParameterError("vertex range out of bounds")
    st = model.device_state()
    ref = np.asarray(ref, dtype=np.float64).reshape(3)
    if out is None:
        out = torch.empty(v1 - v0, dtype=torch.float32, device=st.device)
    else:
        _check_out(out, torch.float32, (v1 - v0,), st.device)
    N.call("ndf_query_grid", st.desc_ref, float(ref[0]), float(ref[1]), float(ref[2]),
           1 if role == ROLE_MU else 0, dims[0], dims[1], dims[2], v0, v1,
           N.PREC[model.spec.precision], out.data_ptr(),
           torch.cuda.current_stream(st.device).cuda_stream)
    if clamp:
        if not out.is_cuda:
            torch.cuda.current_stream(st.device).synchronize()
        out.clamp_(-1.0, 1.0)
    return out


def _check_out(out, dtype, shape, device) -> None:
    """Caller-supplied output buffers: the kernels write exactly ``shape`` elements
    through the raw pointer, so anything else is refused before the launch."""
    import torch
    if not isinstance(out, torch.Tensor) or out.dtype != dtype:
        raise ParameterError(f"out must be a {dtype} tensor")
    if len(shape) == 1:
        if not out.is_contiguous() or out.numel() < shape[0]:
            raise ParameterError(f"out must be contiguous with >= {shape[0]} elements")
    else:
        if (out.dim() != 2 or out.shape[0] < shape[0] or out.shape[1] < shape[1]
                or out.stride(1) != 1):
            raise ParameterError(f"out must be a row-major {shape[0]} x {shape[1]} (or larger) "
                                 "tensor")
    if out.is_cuda:
        if out.device != device:
            raise ParameterError(f"out is on {out.device}, the model on {device}")
    elif not out.is_pinned():
        raise ParameterError("out must be CUDA memory or pinned host memory")


def reconstruct_field(model: NdfModel, ref, role: str = ROLE_MU, dims=(64, 64, 64),
                      batch_size: int = DEFAULT_QUERY_BATCH, clamp: bool = False) -> FieldGrid:
    """service.py:46-84 -- dependence field of ``ref`` over the output grid.  ``model``
    is this package's NdfModel or the reference's own (converted once, as_model)."""
    _check_role(role)
    model = as_model(model)
    if batch_size < 1:
        raise ParameterError("batch_size must be >= 1")
    dims = _check_dims(dims)
    return FieldGrid(dims, _query_to_host(model, ref, role, dims, clamp))


def _query_to_host(model: NdfModel, ref, role, dims, clamp) -> np.ndarray:
    """Query straight into page-locked host memory: the kernel's output stores go over
    PCIe as it runs (ndf_query_grid accepts pinned host pointers), so there is no
    separate D2H copy after it -- measured on B200 that copy was 0.135 ms of a
    0.47 ms end-to-end query; splitting the launch to overlap it lost more than it
    saved.  One stream sync; the array owns the pinned block.  (Arguments are already
    checked by reconstruct_field; this is the per-call host path, kept lean.)"""
    import torch
    st = model.device_state()                    # raises DeviceError without a GPU
    ref = np.asarray(ref, dtype=np.float64).reshape(3)
    V = dims[0] * dims[1] * dims[2]
    host = torch.empty(V, dtype=torch.float32, pin_memory=True)
    stream = torch.cuda.current_stream(st.device)
    N.call("ndf_query_grid", st.desc_ref, float(ref[0]), float(ref[1]), float(ref[2]),
           1 if role == ROLE_MU else 0, dims[0], dims[1], dims[2], 0, V,
           N.PREC[model.spec.precision], host.data_ptr(), stream.cuda_stream)
    stream.synchronize()
    arr = host.numpy()
    if clamp:
        np.clip(arr, -1.0, 1.0, out=arr)
    return arr


def to_host(t) -> np.ndarray:
    """D2H through pinned memory (torch's caching host allocator): one async copy,
    one stream sync; the returned array owns the pinned block until freed."""
    import torch
    host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    host.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return host.numpy()


def difference_field(model: NdfModel, ref_a, ref_b, dims, role: str = ROLE_MU,
                     batch_size: int = DEFAULT_QUERY_BATCH) -> FieldGrid:
    """service.py:87-94 -- reconstruct(ref_a) - reconstruct(ref_b), elementwise (fp32)."""
    return difference_response(model, ref_a, ref_b, dims, role, batch_size).grid()


# ---- binary data plane (/api/reconstruct, /api/diff without the HTTP layer) ----------

@dataclass
class FieldResponse:
    """What ``/api/reconstruct`` and ``/api/diff`` send (service.py:392-396): the field as
    little-endian fp32 bytes (x fastest) and the ``_field_headers`` of service.py:352-360.
    ``body`` is a zero-copy view of the page-locked buffer the export kernel wrote;
    ``content()`` is the ``bytes`` an HTTP layer would send."""
    dims: tuple
    body: memoryview
    headers: dict
    media_type: str = "application/octet-stream"
    _values: np.ndarray | None = None

    def content(self) -> bytes:
        return bytes(self.body)

    def grid(self) -> FieldGrid:
        return FieldGrid(self.dims, self._values)


def _key_to_float(key: int) -> float:
    bits = key ^ 0x80000000 if key & 0x80000000 else (~key) & 0xFFFFFFFF
    return float(np.array([bits], dtype=np.uint32).view(np.float32)[0])


def _export(dims, fa, fb, clamp: bool) -> FieldResponse:
    """One ndf_field_export launch: body (a or a - b, clipped if clamp) into pinned host
    memory plus the min / max keys; one stream sync."""
    import torch
    V = dims[0] * dims[1] * dims[2]
    host = torch.empty(V, dtype=torch.float32, pin_memory=True)
    stats = torch.empty(3, dtype=torch.int32, device=fa.device)
    stream = torch.cuda.current_stream(fa.device)
    N.call("ndf_field_export", fa.data_ptr(), 0 if fb is None else fb.data_ptr(), V,
           host.data_ptr(), stats.data_ptr(), 1 if clamp else 0, stream.cuda_stream)
    st = stats.cpu().numpy().view(np.uint32)          # syncs the stream
    values = host.numpy()
    if V == 0:
        lo = hi = 0.0
    elif st[2]:
        lo = hi = float("nan")                        # np.min / np.max propagate NaN
    else:
        lo, hi = _key_to_float(int(st[0])), _key_to_float(int(st[1]))
    return FieldResponse(dims, memoryview(values).cast("B"), field_headers(dims, lo, hi),
                         _values=values)


def field_headers(dims, lo: float, hi: float) -> dict:
    """``_field_headers`` (service.py:352-360) from the value range."""
    x, y, z = dims
    return {"X-Dims": f"{x},{y},{z}", "X-Value-Min": repr(float(lo)),
            "X-Value-Max": repr(float(hi))}


def reconstruct_response(model: NdfModel, ref, role: str = ROLE_MU, dims=(64, 64, 64),
                         batch_size: int = DEFAULT_QUERY_BATCH,
                         clamp: bool = False) -> FieldResponse:
    """``/api/reconstruct`` (service.py:406-410 + ``_binary`` :392-396): ONE query launch
    (ndf_query_grid_stats) stores the body straight into page-locked host memory and
    reduces the header's value range in its epilogue; the clamp is applied as in
    reconstruct_field (np.clip), and min / max of clipped values are the clipped range."""
    import torch
    _check_role(role)
    model = as_model(model)
    if batch_size < 1:
        raise ParameterError("batch_size must be >= 1")
    dims = _check_dims(dims)
    st = model.device_state()
    ref = np.asarray(ref, dtype=np.float64).reshape(3)
    V = dims[0] * dims[1] * dims[2]
    host = torch.empty(V, dtype=torch.float32, pin_memory=True)
    stats = torch.empty(3, dtype=torch.int32, device=st.device)
    stream = torch.cuda.current_stream(st.device)
    N.call("ndf_query_grid_stats", st.desc_ref, float(ref[0]), float(ref[1]), float(ref[2]),
           1 if role == ROLE_MU else 0, dims[0], dims[1], dims[2], 0, V,
           N.PREC[model.spec.precision], host.data_ptr(), stats.data_ptr(), stream.cuda_stream)
    k = stats.cpu().numpy().view(np.uint32)           # syncs the stream
    values = host.numpy()
    if k[2]:
        lo = hi = float("nan")
    else:
        lo, hi = _key_to_float(int(k[0])), _key_to_float(int(k[1]))
    if clamp:                                          # clip is monotone: range clips too
        np.clip(values, -1.0, 1.0, out=values)
        if not k[2]:
            lo, hi = min(max(lo, -1.0), 1.0), min(max(hi, -1.0), 1.0)
    return FieldResponse(dims, memoryview(values).cast("B"), field_headers(dims, lo, hi),
                         _values=values)


def difference_response(model: NdfModel, ref_a, ref_b, dims, role: str = ROLE_MU,
                        batch_size: int = DEFAULT_QUERY_BATCH) -> FieldResponse:
    """``/api/diff`` (service.py:412-416): two queries into HBM, their fp32 difference
    (difference_field, service.py:87-94) formed inside the export kernel."""
    _check_role(role)
    model = as_model(model)
    dims = _check_dims(dims)
    fa = reconstruct_field_device(model, ref_a, role, dims)
    fb = reconstruct_field_device(model, ref_b, role, dims)
    return _export(dims, fa, fb, False)


PSNR_CAP_DB = 200.0                 # training.py:30


def psnr(predicted, truth, peak: float | None = None) -> float:
    """training.py:162-180 -- 10 log10(peak^2 / MSE) in dB, capped at PSNR_CAP_DB; ``peak``
    defaults to the truth's value range (floored at 1e-6); exact matches return the cap."""
    predicted = np.asarray(predicted, dtype=np.float64).ravel()
    truth = np.asarray(truth, dtype=np.float64).ravel()
    if predicted.size == 0 or predicted.shape != truth.shape:
        raise ParameterError("need equally sized, non-empty inputs")
    if peak is None:
        peak = max(float(np.ptp(truth)), 1e-6)
    if not peak > 0:
        raise ParameterError(f"peak must be positive, got {peak}")
    mse = float(np.mean((predicted - truth) ** 2))
    if mse == 0.0:
        return PSNR_CAP_DB
    return min(10.0 * np.log10(peak * peak / mse), PSNR_CAP_DB)


@dataclass
class ComparisonResult:
    """service.py:128-132."""
    psnr_db: float
    max_abs_err: float
    error_field: FieldGrid


def compare_to_ground_truth(model: NdfModel, field_obj, measure: CorrelationMeasure, ref,
                            dims, role: str = ROLE_MU, workers: int = 1) -> ComparisonResult:
    """service.py:135-155 -- the NDF reconstruction against the direct estimator field on
    the same grid (the paper's evaluation): both fields are computed on the GPU
    (ground_truth_field: one streaming Pearson pass or the KSG kernel; reconstruct_field:
    the query kernels), the error field and PSNR on the host as the reference does."""
    _check_role(role)
    model = as_model(model)
    var_mu, var_nu = model.spec.var_mu, model.spec.var_nu
    if role == ROLE_MU:
        truth = ground_truth_field(field_obj, measure, var_mu, var_nu, ref, dims, workers=workers)
    else:
        truth = ground_truth_field(field_obj, measure, var_nu, var_mu, ref, dims, workers=workers)
    recon = reconstruct_field(model, ref, role, dims)
    err = recon.values.astype(np.float64) - truth.values.astype(np.float64)
    return ComparisonResult(
        psnr_db=psnr(recon.values, truth.values),
        max_abs_err=float(np.max(np.abs(err))) if err.size else 0.0,
        error_field=FieldGrid(dims, err.astype(np.float32)),
    )


def matrix_reconstruct(models: list, variables: list, ref, dims,
                       batch_size: int = DEFAULT_QUERY_BATCH) -> list:
    """service.py:97-125 -- all d*d fields for one reference point, row-major."""
    models = [as_model(m) for m in models]
    by_pair = {(m.spec.var_mu, m.spec.var_nu): m for m in models}
    missing = []
    for i, vi in enumerate(variables):
        for vj in variables[i:]:
            if (vi, vj) not in by_pair and (vj, vi) not in by_pair:
                missing.append((vi, vj))
    if missing:
        raise NotFoundError(f"no model for variable pairs: {missing}")
    cells = []
    for vi in variables:
        for vj in variables:
            if (vi, vj) in by_pair:
                cells.append(reconstruct_field(by_pair[(vi, vj)], ref, ROLE_NU, dims, batch_size))
            else:
                cells.append(reconstruct_field(by_pair[(vj, vi)], ref, ROLE_MU, dims, batch_size))
    return cells


@dataclass
class BenchmarkReport:
    dims: tuple
    repetitions: int
    ndf_seconds: float
    pearson_seconds: float
    mi_seconds: float
    mi_measured_points: int
    mi_extrapolated: bool
    robust: bool

    def speedup_vs_pearson(self) -> float:
        return self.pearson_seconds / self.ndf_seconds

    def speedup_vs_mi(self) -> float:
        return self.mi_seconds / self.ndf_seconds

    def to_csv(self, path) -> None:
        with open(path, "w") as fh:
            fh.write("method,seconds,extrapolated,points\n")
            n = self.dims[0] * self.dims[1] * self.dims[2]
            fh.write(f"ndf,{self.ndf_seconds:.6f},false,{n}\n")
            fh.write(f"pearson,{self.pearson_seconds:.6f},false,{n}\n")
            fh.write(f"ksg_mi,{self.mi_seconds:.6f},"
                     f"{'true' if self.mi_extrapolated else 'false'},{self.mi_measured_points}\n")


def benchmark(model: NdfModel, field_obj, ref, dims, repetitions: int = 3, k: int = 3,
              mi_points: int = 1024) -> BenchmarkReport:
    """service.py:186-220 -- median wall clock of NDF vs direct estimators (GPU)."""
    import torch
    model = as_model(model)
    if repetitions < 1:
        raise ParameterError("repetitions must be >= 1")
    dims = _check_dims(dims)
    n_points = dims[0] * dims[1] * dims[2]
    mi_points = min(mi_points, n_points)
    var = model.spec.var_mu

    def timed(fn):
        samples = []
        for _ in range(repetitions):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            samples.append(time.perf_counter() - t0)
        return statistics.median(samples)

    ndf_s = timed(lambda: reconstruct_field(model, ref, ROLE_MU, dims))
    pearson_s = timed(lambda: ground_truth_field(field_obj, CorrelationMeasure("pearson"), var,
                                                 var, ref, dims))
    mi_measure = CorrelationMeasure("ksg_mi", ksg_k=k)
    mi_sub = timed(lambda: ground_truth_field(field_obj, mi_measure, var, var, ref,
                                              (mi_points, 1, 1)))
    mi_s = mi_sub * (n_points / mi_points)
    return BenchmarkReport(dims, repetitions, ndf_s, pearson_s, mi_s, mi_points,
                           mi_points < n_points, repetitions > 1)


def reconstruct_multi_device(model: NdfModel, refs, role: str = ROLE_MU, dims=(64, 64, 64),
                             v0: int = 0, v1: int | None = None, out=None):
    """Dependence cube of several reference points: fp16 CUDA tensor (n_ref, v1 - v0).

    BASELINE config 3 (64 references x 1.76 M vertices per model).  The batched
    form of the reference's per-reference loop (service.py:97-125), one launch:
    sum_absdiff models run the ping-pong kernel over reference x vertex tiles with
    per-reference feature tables, the other merges embed each query vertex once and
    reuse it for every reference.  Row r equals the single-reference query of
    refs[r] rounded to fp16, bit for bit.
    """
    import torch
    _check_role(role)
    model = as_model(model)
    dims = _check_dims(dims)
    V = dims[0] * dims[1] * dims[2]
    v1 = V if v1 is None else int(v1)
    if not 0 <= v0 <= v1 <= V:
        raise ParameterError("vertex range out of bounds")
    if model.spec.precision not in ("bf16", "fp16"):
        raise ParameterError("multi-reference queries run on the tensor-core path "
                             "(precision 'fp16' or 'bf16')")
    st = model.device_state()
    refs_np = np.ascontiguousarray(np.asarray(refs, dtype=np.float64).reshape(-1, 3))
    n_ref = refs_np.shape[0]
    drefs = torch.from_numpy(refs_np).to(st.device)
    if out is None:
        out = torch.empty((n_ref, v1 - v0), dtype=torch.float16, device=st.device)
    else:
        _check_out(out, torch.float16, (n_ref, v1 - v0), st.device)
    N.call("ndf_query_grid_multi", ctypes_ref(st.desc), N.ptr(drefs), n_ref,
           1 if role == ROLE_MU else 0, dims[0], dims[1], dims[2], v0, v1, N.ptr(out),
           out.stride(0), N.stream_handle(st.device))
    return out


def forward(model, p_mu, p_nu, exact: bool = True) -> np.ndarray:
    """NdfModel.forward (model.py:179-189) for this package's models or the reference's
    own (as_model): batched dependence estimates, shape (B,) float32."""
    return as_model(model).forward(p_mu, p_nu, exact)
