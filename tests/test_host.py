"""CPU-only tests: C-ABI library loads and exports every declared symbol, host
logic (specs, containers, IO, error mapping) mirrors the reference."""

import os
import re

import numpy as np
import pytest

import paper_2307_02203_b200 as ndf
from paper_2307_02203_b200 import _native as N
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

HEADER = os.path.join(ROOT, "include", "ndf_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ndf_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    if not os.path.exists(N.LIB_PATH):
        from paper_2307_02203_b200 import build
        build.build()
    lib = N.load_library()
    syms = declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(N.SIGNATURES), set(syms) ^ set(N.SIGNATURES)
    assert lib.ndf_abi_version() == N.NDF_ABI_VERSION == 3


def test_status_mapping():
    N.load_library()
    with pytest.raises(ndf.ParameterError):
        N.check(1)
    with pytest.raises(ndf.ShapeError):
        N.check(2)
    with pytest.raises(ndf.ConfigError):
        N.check(5)
    with pytest.raises(ndf.DeviceError):
        N.check(4)
    N.check(0)


def test_model_desc_layout_matches_c_header(tmp_path):
    """The ctypes mirror of ndf_model_desc has the C compiler's size and offsets."""
    import ctypes
    import shutil
    import subprocess
    gcc = shutil.which("gcc") or shutil.which("cc")
    if gcc is None:
        pytest.skip("no C compiler")
    fields = [f for f, _ in N.ModelDesc._fields_]
    src = tmp_path / "layout.c"
    src.write_text("#include <stdio.h>\n#include <stddef.h>\n#include \"ndf_b200.h\"\n"
                   "int main(void){printf(\"%zu\\n\", sizeof(ndf_model_desc));"
                   + "".join(f'printf("%zu\\n", offsetof(ndf_model_desc, {f}));' for f in fields)
                   + "return 0;}\n")
    exe = tmp_path / "layout"
    subprocess.run([gcc, "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    vals = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                           check=True).stdout.split()]
    assert vals[0] == ctypes.sizeof(N.ModelDesc)
    for f, off in zip(fields, vals[1:]):
        assert getattr(N.ModelDesc, f).offset == off, f


def test_modelspec_baseline_shapes():
    spec = ndf.ModelSpec.baseline((250, 352, 20), 4)
    assert spec.latent_resolution == (63, 88, 5)
    assert spec.embed_dim == 55
    assert spec.decoder_widths() == [110, 128, 128, 128, 1]
    assert spec.head_kind == "tanh"
    spec0 = ndf.ModelSpec.baseline((32, 44, 4), 8)
    assert spec0.latent_resolution == (4, 6, 2)
    assert ndf.ModelSpec(measure_kind="ksg_mi").head_kind == "softplus"
    with pytest.raises(ndf.ConfigError):
        ndf.ModelSpec(merge="average")
    # reference family (encoders / HashGrid): exact fp32 path only
    ndf.ModelSpec(encoder_layers=2).check_gpu_supported()
    ndf.ModelSpec.reference_default().check_gpu_supported()
    with pytest.raises(ndf.ConfigError):
        ndf.ModelSpec(encoder_layers=2, precision="fp16").check_gpu_supported()
    with pytest.raises(ndf.ConfigError):
        ndf.ModelSpec.reference_default(levels=17).check_gpu_supported()
    with pytest.raises(ndf.ConfigError):
        ndf.ModelSpec(var_mu="a", var_nu="b", shared_encoder=True)


def test_build_matches_oracle_rng_order():
    from oracle import ndf_oracle as O
    spec = ndf.ModelSpec.baseline((32, 44, 4), 8)
    m = ndf.NdfModel.build(spec, seed=0)
    o = O.build_model((32, 44, 4), factor=8, seed=0)
    assert np.array_equal(m.grid_mu, o.grid_mu)
    for a, b in zip(m.weights, o.weights):
        assert np.array_equal(a, b)


def test_ndfm_roundtrip(tmp_path):
    spec = ndf.ModelSpec.baseline((32, 44, 4), 8, shared_encoder=False, var_mu="a", var_nu="b")
    m = ndf.NdfModel.build(spec, seed=4)
    p = tmp_path / "m.ndfm"
    ndf.save_model(m, p)
    m2 = ndf.load_model(p)
    assert m2.spec == m.spec
    for a, b in zip(m.parameters(), m2.parameters()):
        assert np.array_equal(a, b)


def test_load_reference_ndfm(tmp_path):
    """A reference-format NDFM (encoder-less, one dense level) loads as a GPU model."""
    import json
    import struct
    rng = np.random.default_rng(0)
    header = dict(var_mu="v", var_nu="v", measure_kind="pearson", merge="add",
                  shared_encoder=True, fourier_octaves=6, levels=1, base_resolution=4,
                  growth=2.0, log2_table_size=6, features_per_level=16, encoder_layers=0,
                  decoder_layers=2, channels=8, encoder_widths=[55], decoder_widths=[55, 8, 1])
    table = rng.uniform(-1, 1, (1, 64, 16)).astype(np.float32)
    w0 = rng.standard_normal((55, 8)).astype(np.float32)
    b0 = rng.standard_normal(8).astype(np.float32)
    w1 = rng.standard_normal((8, 1)).astype(np.float32)
    b1 = rng.standard_normal(1).astype(np.float32)
    raw = json.dumps(header, sort_keys=True).encode()
    p = tmp_path / "ref.ndfm"
    with open(p, "wb") as fh:
        fh.write(b"NDFM" + struct.pack("<2I", 1, len(raw)) + raw)
        for a in (table, w0, b0, w1, b1):
            fh.write(a.tobytes())
    m = ndf.load_model(p)
    assert m.spec.activation == "snake_alt" and m.spec.head_kind == "linear"
    assert np.array_equal(m.grid_mu, table[0].reshape(4, 4, 4, 16))


def test_ndfe_roundtrip_and_errors(tmp_path):
    rng = np.random.default_rng(7)
    vals = rng.standard_normal((2, 9, 4, 5, 6)).astype(np.float32)
    f = ndf.EnsembleField(ndf.GridDomain(6, 5, 4), ("a", "b"), vals)
    p = tmp_path / "e.ndfe"
    ndf.save_ensemble(f, p)
    g = ndf.load_ensemble(p)
    assert g.variables == ("a", "b") and np.array_equal(g.values, vals)
    bad = tmp_path / "bad.ndfe"
    bad.write_bytes(b"NOPE" + b"\0" * 24)
    with pytest.raises(ndf.FormatError):
        ndf.load_ensemble(bad)
    trunc = tmp_path / "t.ndfe"
    trunc.write_bytes(p.read_bytes()[:-4])
    with pytest.raises(ndf.CorruptFileError):
        ndf.load_ensemble(trunc)
    with pytest.raises(ndf.UnknownVariableError):
        f.member_grids("zz")


def test_ndfe_bytes_identical_to_reference_writer(tmp_path):
    """Our NDFE writer produces the reference container byte for byte (ensemble.py:283-294)."""
    import struct
    vals = np.arange(2 * 3 * 2 * 2 * 2, dtype=np.float32).reshape(1, 3, 2, 2, 2 * 2)[:, :, :, :, :2]
    vals = np.ascontiguousarray(vals)
    f = ndf.EnsembleField(ndf.GridDomain(2, 2, 2), ("v",), vals)
    p = tmp_path / "x.ndfe"
    ndf.save_ensemble(f, p)
    want = b"NDFE" + struct.pack("<6I", 1, 2, 2, 2, 3, 1) + struct.pack("<H", 1) + b"v" + \
        vals.astype("<f4").tobytes()
    assert p.read_bytes() == want


def test_fieldgrid_and_ndfg(tmp_path):
    rng = np.random.default_rng(3)
    grid = ndf.FieldGrid((4, 3, 2), rng.standard_normal(24).astype(np.float32))
    p = tmp_path / "f.ndfg"
    ndf.save_field_grid(grid, p)
    g = ndf.load_field_grid(p)
    assert g.dims == (4, 3, 2) and np.array_equal(g.values, grid.values)
    with pytest.raises(ndf.ParameterError):
        ndf.FieldGrid((0, 2, 2), np.zeros(0, dtype=np.float32))
    with pytest.raises(ndf.ParameterError):
        ndf.FieldGrid((2, 2, 2), np.zeros(7, dtype=np.float32))


def test_digamma_matches_reference_golden(golden):
    g = golden("ksg")
    assert np.array_equal(ndf.digamma(np.arange(1, 2001, dtype=np.float64)), g["psi"])
    with pytest.raises(ndf.ParameterError):
        ndf.digamma(0.0)


def test_measure_validation():
    with pytest.raises(ndf.ParameterError):
        ndf.CorrelationMeasure("spearman")
    with pytest.raises(ndf.ParameterError):
        ndf.CorrelationMeasure("ksg_mi", ksg_k=0)
    assert ndf.gaussian_mi_analytic(0.5) == pytest.approx(0.143841, abs=1e-6)
    with pytest.raises(ndf.ParameterError):
        ndf.gaussian_mi_analytic(1.0)


def test_compute_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    spec = ndf.ModelSpec(grid_resolution=(3, 3, 3))
    m = ndf.NdfModel.build(spec, seed=1)
    with pytest.raises(ndf.DeviceError):
        ndf.reconstruct_field(m, (0, 0, 0), ndf.ROLE_MU, (4, 4, 4))
    with pytest.raises(ndf.DeviceError):
        ndf.ksg_mi(np.arange(10.0), np.arange(10.0) ** 2, 3)


def test_workload_pairs_and_refs():
    from paper_2307_02203_b200 import workloads as W
    w = W.CONFIGS[4]
    a, b = W.pair_list(w, count=1000)
    assert a.shape == b.shape == (1000,)
    assert a.min() >= 0 and max(a.max(), b.max()) < w.n_vertices
    nx, ny = w.dims[0], w.dims[1]
    near = slice(500, 1000)
    for arr_a, arr_b in [(a[near], b[near])]:
        d = np.abs((arr_a % nx) - (arr_b % nx))
        assert d.max() <= 16
    refs = W.reference_vertices(W.CONFIGS[3])
    assert refs.shape == (64,)


def test_reference_default_build_matches_reference_rng(golden):
    """NdfModel.build(reference default, seed) draws the reference's parameters
    (model.py:131-142): per-array sums / first elements from the golden fixture, and
    bit-for-bit against the importable reference where it exists (build container)."""
    g = golden("ndf_refdefault")
    m = ndf.NdfModel.build(ndf.ModelSpec.reference_default(), seed=0)
    params = m.parameters()
    assert len(params) == len(g["default_param_sums"])
    for p, s, f in zip(params, g["default_param_sums"], g["default_param_first"]):
        assert float(np.sum(p, dtype=np.float64)) == s
        assert float(p.ravel()[0]) == f
    ref_src = "/root/reference/pkg/src"
    if not os.path.isdir(ref_src):
        return
    import sys
    sys.path.insert(0, ref_src)
    try:
        from ndf.model import ModelSpec as RefSpec, NdfModel as RefModel
    finally:
        sys.path.remove(ref_src)
    r = RefModel.build(RefSpec(), seed=0)
    for a, b in zip(params, r.parameters()):
        assert np.array_equal(a, b)


def test_reference_ndfm_with_hashgrid_and_encoders(tmp_path, golden):
    """An NDFM written in the reference layout for its default family (HashGrid tables,
    encoders, decoder) loads unchanged and round-trips through save_model."""
    import json
    import struct
    import refdefault as R
    g = golden("ndf_refdefault")
    m = R.golden_case(g, "add2")
    spec = m.spec
    header = {k: getattr(spec, k) for k in ("var_mu", "var_nu", "measure_kind", "merge",
                                             "fourier_octaves", "levels", "base_resolution",
                                             "growth", "log2_table_size", "features_per_level",
                                             "encoder_layers", "decoder_layers", "channels")}
    header.update(shared_encoder=spec.shared, encoder_widths=spec.encoder_widths(),
                  decoder_widths=spec.decoder_widths())
    raw = json.dumps(header, sort_keys=True).encode()
    p = tmp_path / "ref.ndfm"
    with open(p, "wb") as fh:
        fh.write(b"NDFM" + struct.pack("<2I", 1, len(raw)) + raw)
        for a in m.parameters():
            fh.write(np.ascontiguousarray(a, "<f4").tobytes())
    m2 = ndf.load_model(p)
    assert m2.spec.hash_grid and m2.spec.activation == "snake_alt" and m2.spec.head_kind == "linear"
    assert len(m2.parameters()) == len(m.parameters())
    for a, b in zip(m.parameters(), m2.parameters()):
        assert np.array_equal(a, b)
    q = tmp_path / "ours.ndfm"
    ndf.save_model(m2, q)
    m3 = ndf.load_model(q)
    assert m3.spec == m2.spec
    for a, b in zip(m2.parameters(), m3.parameters()):
        assert np.array_equal(a, b)


def test_bench_reference_arm_contract():
    """bench.py --impl reference prints one JSON line with the contract's keys (CPU)."""
    import json
    import subprocess
    import sys
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0", "--ref-sample", "2048"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "cpu_baseline", "e2e", "config"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
