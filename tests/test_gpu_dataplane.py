"""Binary data plane of /api/reconstruct and /api/diff (service.py:392-416) on the GPU:
reconstruct_response / difference_response against reconstruct_field and the reference's
header formula (service.py:352-360: repr of float(values.min()) / float(values.max())),
and ndf_field_export's edge cases (tails, misalignment, NaN, clamp, empty)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2307_02203_b200 as ndf  # noqa: E402
from paper_2307_02203_b200 import _native as N  # noqa: E402
from paper_2307_02203_b200 import service as S  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402


def _ref_headers(dims, values):
    """service.py:352-360 restated (the reference is not on the GPU box; the CPU test
    tests/test_dropin.py pins field_headers to the reference's own function)."""
    lo = float(values.min()) if values.size else 0.0
    hi = float(values.max()) if values.size else 0.0
    x, y, z = dims
    return {"X-Dims": f"{x},{y},{z}", "X-Value-Min": repr(lo), "X-Value-Max": repr(hi)}


@pytest.fixture(scope="module")
def model():
    w = W.CONFIGS[0]
    return w, W.build_model(w, seed=0, grid_init=1.0)


def _variant(base, kind):
    if kind == "classic":          # merge outside the x3 / ping-pong family -> query_tc_kernel
        spec = base.spec
        m = ndf.NdfModel.build(ndf.ModelSpec(**{**spec.__dict__, "merge": "concat"}), seed=4)
        return m.with_precision("bf16")
    return base.with_precision(kind)


@pytest.mark.parametrize("prec", ["fp32", "bf16", "fp16", "classic"])
def test_reconstruct_response_body_and_headers(model, prec):
    """ndf_query_grid_stats: the range reduced inside each query kernel (f32, x3,
    ping-pong, classic) equals NumPy's min / max of the body."""
    w, base = model
    m = _variant(base, prec)
    for clamp in (False, True):
        grid = ndf.reconstruct_field(m, w.ref_position(), ndf.ROLE_MU, w.dims, clamp=clamp)
        resp = ndf.reconstruct_response(m, w.ref_position(), ndf.ROLE_MU, w.dims, clamp=clamp)
        assert resp.media_type == "application/octet-stream"
        assert resp.content() == grid.values.astype("<f4").tobytes()
        assert resp.headers == _ref_headers(w.dims, grid.values)
        assert resp.grid().dims == grid.dims


def test_difference_response_and_field(model):
    w, m = model
    a, b = (0.11, -0.4, 0.7), (-0.6, 0.25, -0.1)
    fa = ndf.reconstruct_field(m, a, ndf.ROLE_NU, w.dims).values
    fb = ndf.reconstruct_field(m, b, ndf.ROLE_NU, w.dims).values
    want = fa - fb
    resp = ndf.difference_response(m, a, b, w.dims, ndf.ROLE_NU)
    assert resp.content() == want.astype("<f4").tobytes()
    assert resp.headers == _ref_headers(w.dims, want)
    diff = ndf.difference_field(m, a, b, w.dims, ndf.ROLE_NU)
    assert np.array_equal(diff.values, want)


def _export(a, b=None, clamp=False, dims=None):
    dims = dims or (a.numel(), 1, 1)
    return S._export(dims, a, b, clamp)


def test_field_export_edges():
    dev = torch.device("cuda")
    rng = np.random.default_rng(0)
    base = torch.from_numpy(rng.standard_normal(4099).astype(np.float32) * 3).to(dev)
    for off in (0, 1, 2, 3):                          # scalar path for misaligned views
        for n in (1, 3, 4, 5, 1024, 4095 - off):
            a = base[off:off + n]
            b = base[-n:]
            va, vb = a.cpu().numpy(), b.cpu().numpy()
            r = _export(a)
            assert r.content() == va.tobytes()
            assert r.headers == _ref_headers((n, 1, 1), va)
            r = _export(a, b, clamp=True)
            want = np.clip(va - vb, -1.0, 1.0)
            assert r.content() == want.astype("<f4").tobytes()
            assert r.headers == _ref_headers((n, 1, 1), want)
    # NaN anywhere: body keeps it, headers say nan like np.min / np.max
    a = base[:4096].clone()
    a[1234] = float("nan")
    r = _export(a, clamp=True)
    got = np.frombuffer(r.content(), dtype="<f4")
    assert np.isnan(got[1234]) and np.isnan(got).sum() == 1
    assert r.headers["X-Value-Min"] == "nan" and r.headers["X-Value-Max"] == "nan"
    # empty field
    r = _export(base[:0], dims=(0, 4, 4))
    assert r.content() == b"" and r.headers == _ref_headers((0, 4, 4), np.zeros(0, np.float32))


def test_field_export_counts_one_launch():
    a = torch.randn(1 << 20, device="cuda")
    lib = N.load_library()
    lib.ndf_launch_count(1)
    _export(a)
    assert lib.ndf_launch_count(1) == 1
