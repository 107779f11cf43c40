"""GPU parity of the ground-truth estimators (Pearson K3, KSG K4, sampling).

KSG neighbour / marginal counts must be bit-exact; Pearson fp32 fields within
1e-5 absolute (BASELINE north_star).  Golden values come from the unmodified
reference (tests/golden/make_golden.py).
"""

import logging

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2307_02203_b200 as ndf  # noqa: E402
from oracle import ndf_oracle as O  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402


def field_from(grids):
    nz, ny, nx = grids.shape[1:]
    return ndf.EnsembleField(ndf.GridDomain(nx, ny, nz), ("v",), grids[None])


# ---- sampling ----------------------------------------------------------------

def test_sample_many_bitwise(golden):
    g = golden("pearson")
    got = ndf.sample_many(field_from(g["field"]), "v", g["sample_pos"])
    assert np.array_equal(got, g["sample_out"])


# ---- Pearson -------------------------------------------------------------------

def test_pearson_known_answers():
    # reference tests/test_measures.py:51-98
    assert ndf.pearson([1, 2, 3], [2, 4, 6]) == 1.0
    assert ndf.pearson([1, 2, 3], [3, 2, 1]) == -1.0
    assert ndf.pearson([1, 2, 3, 4], [1, 3, 2, 4]) == pytest.approx(0.8, abs=1e-15)
    a = np.random.default_rng(5).standard_normal(37)
    assert ndf.pearson(a, a.copy()) == 1.0
    with pytest.raises(ndf.DegenerateSampleError):
        ndf.pearson([1.0, 1.0, 1.0], [1, 2, 3])
    with pytest.raises(ndf.ParameterError):
        ndf.pearson([1, 2], [1, 2, 3])
    assert np.isnan(ndf.pearson_rowwise(np.ones((2, 5)), np.arange(10.0).reshape(2, 5))).all()


def test_pearson_rowwise_golden(golden):
    g = golden("pearson")
    got = ndf.pearson_rowwise(g["rw_a"], g["rw_b"])
    want = g["rw_out"]
    assert np.array_equal(np.isnan(got), np.isnan(want))
    ok = ~np.isnan(want)
    assert np.max(np.abs(got[ok] - want[ok])) <= 1e-12
    assert got[3] == 1.0
    got = ndf.pearson_against(g["rw_a"][0], g["rw_b"])
    want = g["against_out"]
    ok = ~np.isnan(want)
    assert np.max(np.abs(got[ok] - want[ok])) <= 1e-12


@pytest.mark.parametrize("name", ["node", "offnode"])
def test_ground_truth_pearson_golden(golden, name, caplog):
    g = golden("pearson")
    dims = tuple(int(d) for d in g[f"gt_{name}_dims"])
    with caplog.at_level(logging.WARNING):
        got = ndf.ground_truth_field(field_from(g["field"]), ndf.CorrelationMeasure("pearson"),
                                     "v", "v", g[f"gt_{name}_ref"], dims).values
    want = g[f"gt_{name}"]
    assert np.max(np.abs(got - want)) <= 1e-5
    if name == "node":
        assert "degenerate" in caplog.text
        assert got[int(np.flatnonzero(want == 0.0)[0])] == 0.0


def test_self_node_exactly_one_and_white_noise_bound():
    # reference tests/test_measures.py:188-201
    w = W.Workload("white", (5, 5, 4), 200, (0.01, 0.01, 0.01), 2, "fp32", "pearson",
                   ref_vertex=(0, 0, 0), seed=3)
    rng = np.random.default_rng(3)
    grids = rng.standard_normal((200, 4, 5, 5)).astype(np.float32)
    f = field_from(grids)
    grid = ndf.ground_truth_field(f, ndf.CorrelationMeasure("pearson"), "v", "v",
                                  (-1.0, -1.0, -1.0), (5, 5, 4))
    assert grid.values[0] == 1.0
    assert np.max(np.abs(grid.values[1:])) < 4.0 / np.sqrt(200)
    del w


def test_degenerate_reference_maps_to_zero(caplog):
    # reference tests/test_measures.py:203-213
    values = np.zeros((1, 3, 2, 2, 2), dtype=np.float32)
    values[0, :, 1] = np.arange(3)[:, None, None]
    f = ndf.EnsembleField(ndf.GridDomain(2, 2, 2), ("v",), values)
    with caplog.at_level(logging.WARNING):
        grid = ndf.ground_truth_field(f, ndf.CorrelationMeasure("pearson"), "v", "v",
                                      (-1.0, -1.0, -1.0), (2, 2, 2))
    assert np.all(grid.values == 0.0)
    assert "degenerate" in caplog.text


def test_c0_ground_truth_pearson_vs_oracle():
    w = W.CONFIGS[0]
    f = W.generate_host(w)
    ref = w.ref_position()
    got = ndf.ground_truth_field(f, ndf.CorrelationMeasure("pearson"), "v", "v", ref, w.dims).values
    want = O.ground_truth_field(f.member_grids("v"), "pearson", ref, w.dims)
    assert np.max(np.abs(got - want)) <= 1e-5
    assert got[w.ref_flat()] == 1.0


def test_pearson_gemv_unaligned_ranges():
    """Vertex ranges that are not multiples of 4 take the scalar path; same values."""
    rng = np.random.default_rng(8)
    grids = rng.standard_normal((64, 3, 7, 11)).astype(np.float32)   # V = 231 (odd)
    f = field_from(grids)
    dev = f.to_device("v")
    full = ndf.ground_truth_field_device(f, ndf.CorrelationMeasure("pearson"), "v", "v",
                                         (0.0, 0.0, 0.0), (11, 7, 3)).cpu().numpy()
    parts = [ndf.ground_truth_field_device(dev, ndf.CorrelationMeasure("pearson"), "v", "v",
                                           (0.0, 0.0, 0.0), (11, 7, 3), a, b).cpu().numpy()
             for a, b in [(0, 5), (5, 130), (130, 231)]]
    assert np.max(np.abs(np.concatenate(parts) - full)) <= 1e-6
    want = O.ground_truth_field(grids, "pearson", (0.0, 0.0, 0.0), (11, 7, 3))
    assert np.max(np.abs(full - want)) <= 1e-5


@pytest.mark.parametrize("M,nz,ny,nx", [(1000, 2, 30, 40), (37, 3, 7, 11), (5, 1, 1, 133)])
def test_zscore_and_gemv_vs_fp64(M, nz, ny, nx):
    """ndf_zscore (the standardised copy Z callers of ndf_pearson_gemv hold) against a
    fp64 two-pass z-score, on the vectorised (V % 4 == 0) and scalar layouts, with
    constant columns (degenerate: Z = 0, norm = 0) and partial ranges; then the GEMV
    over that Z against the oracle's pearson_against (measures.py:84-108)."""
    from paper_2307_02203_b200 import _native as N
    rng = np.random.default_rng(M + nx)
    X = rng.standard_normal((M, nz, ny, nx)).astype(np.float32)
    X[:, 0, 0, 3] = 2.5                     # constant column -> degenerate
    V = nz * ny * nx
    dev = torch.from_numpy(X.reshape(M, V)).cuda()
    Z = torch.full((M, V), 7.0, dtype=torch.float32, device="cuda")
    norm = torch.full((V,), 7.0, dtype=torch.float32, device="cuda")
    s = N.stream_handle(dev.device)
    for a, b in [(0, V // 3 + 1), (V // 3 + 1, V - 2), (V - 2, V)]:   # ragged ranges
        N.call("ndf_zscore", N.ptr(dev), M, V, a, b, N.ptr(Z), N.ptr(norm), s)
    torch.cuda.synchronize()
    x64 = X.reshape(M, V).astype(np.float64)
    c = x64 - x64.mean(axis=0)
    nrm = np.sqrt((c * c).sum(axis=0))
    ok = nrm > 0
    want = np.zeros_like(c)
    want[:, ok] = c[:, ok] / nrm[ok]
    Zh, nh = Z.cpu().numpy(), norm.cpu().numpy()
    assert np.max(np.abs(Zh - want)) <= 1e-6
    assert np.all(Zh[:, ~ok] == 0.0) and np.all(nh[~ok] == 0.0)
    assert np.max(np.abs(nh[ok] - nrm[ok]) / nrm[ok]) <= 1e-6
    ref = 5 if V > 5 else 0
    zref = Z[:, ref].contiguous()
    out = torch.empty(V, dtype=torch.float32, device="cuda")
    N.call("ndf_pearson_gemv", N.ptr(Z), N.ptr(norm), M, V, N.ptr(zref), 0, 0, V, N.ptr(out), s)
    got = out.cpu().numpy()
    pw = O.pearson_against(x64[:, ref], x64.T)
    assert got[ref] == 1.0
    assert np.array_equal(np.isnan(got), ~ok)          # degenerate -> NaN, as pearson_against
    assert np.max(np.abs(got[ok] - pw[ok])) <= 1e-5


# ---- KSG -------------------------------------------------------------------------

def test_ksg_golden_bitwise(golden):
    g = golden("ksg")
    for i in range(int(g["ksg_cases"])):
        a, b, k = g[f"ksg{i}_a"], g[f"ksg{i}_b"], int(g[f"ksg{i}_k"])
        got = ndf.ksg_mi(a, b, k)
        assert got == float(g[f"ksg{i}_mi"]), (i, got, float(g[f"ksg{i}_mi"]))


def test_ksg_counts_bitexact_m1000():
    """Neighbour and marginal counts bit-exact vs the oracle at the BASELINE shape."""
    rng = np.random.default_rng(11)
    B, M, k = 24, 1000, 8
    a = rng.standard_normal(M).astype(np.float32).astype(np.float64)
    rows = []
    for s in range(B):
        x = 0.7 * a + 0.5 * rng.standard_normal(M)
        y = x + 0.5 * x ** 2 + 0.2 * np.sin(3 * x)
        if s % 6 == 0:
            y = np.round(y, 1)               # heavy ties
        rows.append(y.astype(np.float32).astype(np.float64))
    b = np.stack(rows)
    mi, counts = ndf.ksg_rows(a, b, k, return_counts=True)
    for s in range(B):
        _, nx, ny = O.ksg_counts_bruteforce(a, b[s], k)
        assert np.array_equal(counts[s, 0], nx) and np.array_equal(counts[s, 1], ny)
        assert mi[s] == O.ksg_mi(a, b[s], k)


def test_ksg_properties():
    # reference tests/test_measures.py:132-173
    rng = np.random.default_rng(9)
    x = rng.standard_normal(500)
    y = 0.6 * x + 0.8 * rng.standard_normal(500)
    assert ndf.ksg_mi(x, y, 3) == ndf.ksg_mi(y, x, 3)
    a = np.round(rng.standard_normal(500), 1)
    b = np.round(0.8 * a + 0.2 * rng.standard_normal(500), 1)
    assert np.isfinite(ndf.ksg_mi(a, b, 3))
    assert np.isfinite(ndf.ksg_mi(np.zeros(100), rng.standard_normal(100), 3))
    with pytest.raises(ndf.ParameterError):
        ndf.ksg_mi(rng.random(10), rng.random(10), 10)
    with pytest.raises(ndf.ParameterError):
        ndf.ksg_mi(rng.random(10), rng.random(10), 0)
    with pytest.raises(ndf.ParameterError):      # both constant: digamma(0) in the reference
        ndf.ksg_mi(np.zeros(20), np.ones(20), 3)


def test_ksg_gaussian_analytic():
    ests = []
    for s in range(10):
        r = np.random.default_rng(s)
        x = r.standard_normal(2000)
        y = 0.5 * x + np.sqrt(0.75) * r.standard_normal(2000)
        ests.append(ndf.ksg_mi(x, y, 3))
    assert abs(np.mean(ests) - ndf.gaussian_mi_analytic(0.5)) < 0.05


def test_ground_truth_ksg_golden(golden):
    g = golden("ksg")
    dims = tuple(int(d) for d in g["gt_dims"])
    got = ndf.ground_truth_field(field_from(g["field"]),
                                 ndf.CorrelationMeasure("ksg_mi", ksg_k=int(g["gt_k"])),
                                 "v", "v", g["gt_ref"], dims).values
    assert np.array_equal(got, g["gt_mi"])


def test_c0_ground_truth_ksg_offnode_dims_vs_oracle():
    w = W.CONFIGS[0]
    f = W.generate_host(w)
    dims = (7, 5, 3)
    ref = (0.1, -0.2, 0.3)
    got = ndf.ground_truth_field(f, ndf.CorrelationMeasure("ksg_mi", ksg_k=4), "v", "v", ref,
                                 dims).values
    want = O.ground_truth_field(f.member_grids("v"), "ksg_mi", ref, dims, k=4)
    assert np.array_equal(got, want)


def test_c2_shaped_ksg_field_subset_bitexact():
    """Config-2 generator at reduced grid: node-path KSG field vs oracle, bit-exact."""
    w = W.Workload("c2_small", (24, 20, 4), 1000, (8, 8, 2), 4, "bf16", "ksg_mi",
                   nonlinear=True, ref_vertex=(12, 10, 2), seed=2309)
    dev = W.generate_device(w)
    ref = w.ref_position()
    got = ndf.ground_truth_field_device(dev, ndf.CorrelationMeasure("ksg_mi", ksg_k=8), "v", "v",
                                        ref, w.dims).cpu().numpy()
    X = dev.X.cpu().numpy()
    idx = np.random.default_rng(1).integers(0, w.n_vertices, 64)
    want = O.ground_truth_field(X, "ksg_mi", ref, w.dims, k=8, vertices=idx)
    assert np.array_equal(got[idx], want)


@pytest.mark.parametrize("M", [2, 5, 301, 1000, 1024, 1100])
def test_pearson_pairs_layouts(M):
    """ndf_pearson_pairs on the register-resident path (M % 4 == 0, M <= 1024) and the
    two-pass fallback, with a self pair (1.0), a constant row (NaN, measures.py:124-126)
    and an affine copy, against the oracle's pearson_rowwise."""
    from paper_2307_02203_b200 import _native as N
    rng = np.random.default_rng(M)
    V, n = 40, 64
    Xv = rng.standard_normal((V, M)).astype(np.float32)
    Xv[3] = 1.5                                   # constant row
    Xv[4] = Xv[5] * 2.0 + 0.25                    # affine (r ~ 1, not forced)
    pa = rng.integers(0, V, n)
    pb = rng.integers(0, V, n)
    pa[:4] = [7, 3, 4, 9]
    pb[:4] = [7, 8, 5, 3]
    dev = torch.from_numpy(Xv).cuda()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    tpa, tpb = torch.from_numpy(pa).cuda(), torch.from_numpy(pb).cuda()   # kept alive
    N.call("ndf_pearson_pairs", N.ptr(dev), M, V, N.ptr(tpa), N.ptr(tpb), n, N.ptr(out),
           N.stream_handle())
    got = out.cpu().numpy()
    want = O.pearson_rowwise(Xv[pa].astype(np.float64), Xv[pb].astype(np.float64))
    assert got[0] == 1.0
    assert np.array_equal(np.isnan(got), np.isnan(want)) and np.isnan(got[1]) and np.isnan(got[3])
    ok = ~np.isnan(want)
    assert np.max(np.abs(got[ok] - want[ok])) <= 1e-12


def test_pairs_pearson_and_ksg_vs_oracle():
    rng = np.random.default_rng(21)
    grids = rng.standard_normal((300, 4, 6, 8)).astype(np.float32)
    dev = ndf.DeviceEnsemble.from_numpy(grids)
    Xv = dev.vertex_major()
    V = 4 * 6 * 8
    pa = rng.integers(0, V, 100)
    pb = rng.integers(0, V, 100)
    pa[0] = pb[0]                                     # self pair -> 1.0
    from paper_2307_02203_b200 import _native as N
    tpa = torch.from_numpy(pa).cuda()
    tpb = torch.from_numpy(pb).cuda()
    out = torch.empty(100, dtype=torch.float64, device="cuda")
    N.call("ndf_pearson_pairs", N.ptr(Xv), 300, V, N.ptr(tpa), N.ptr(tpb), 100, N.ptr(out),
           N.stream_handle())
    flat = grids.reshape(300, V)
    want = O.pearson_rowwise(flat[:, pa].T, flat[:, pb].T)
    got = out.cpu().numpy()
    assert got[0] == 1.0
    assert np.max(np.abs(got - want)) <= 1e-12
    from paper_2307_02203_b200.measures import _KsgTables
    jit, psi = _KsgTables.get(torch.device("cuda", torch.cuda.current_device()), 300)
    mi = torch.empty(100, dtype=torch.float64, device="cuda")
    cnt = torch.empty((100, 2, 300), dtype=torch.int32, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.call("ndf_ksg_pairs", N.ptr(Xv), 300, V, N.ptr(tpa), N.ptr(tpb), 100, 8, N.ptr(jit),
           N.ptr(psi), _KsgTables.psi_km(8, 300), N.ptr(mi), None, N.ptr(cnt), N.ptr(st),
           N.stream_handle())
    mi = mi.cpu().numpy()
    cnt = cnt.cpu().numpy()
    for p in range(1, 100, 7):
        a = flat[:, pa[p]].astype(np.float64)
        b = flat[:, pb[p]].astype(np.float64)
        _, nx, ny = O.ksg_counts_bruteforce(a, b, 8)
        assert np.array_equal(cnt[p, 0], nx) and np.array_equal(cnt[p, 1], ny)
        assert mi[p] == O.ksg_mi(a, b, 8)


def test_empty_inputs_everywhere():
    """Empty ranges and batches return empty results (no launch, no error) on every
    GPU entry point: query vertex ranges, paired forward, row-wise Pearson, KSG rows,
    ground-truth vertex ranges, bulk pairs."""
    import torch
    spec = ndf.ModelSpec(grid_resolution=(3, 3, 3))
    model = ndf.NdfModel.build(spec, seed=2)
    for prec in ("fp32", "fp16"):
        m = model.with_precision(prec) if prec != "fp32" else model
        out = ndf.reconstruct_field_device(m, (0, 0, 0), ndf.ROLE_MU, (4, 4, 4), 7, 7)
        assert out.numel() == 0
        assert m.forward(np.zeros((0, 3)), np.zeros((0, 3))).shape == (0,)
    assert ndf.pearson_rowwise(np.zeros((0, 5)), np.zeros((0, 5))).shape == (0,)
    mi, cnt = ndf.ksg_rows(np.zeros((0, 20)), np.zeros((0, 20)), 3, return_counts=True)
    assert mi.shape == (0,) and cnt.shape == (0, 2, 20)
    rng = np.random.default_rng(0)
    f = field_from(rng.standard_normal((30, 3, 4, 5)).astype(np.float32))
    for kind in ("pearson", "ksg_mi"):
        meas = ndf.CorrelationMeasure(kind, ksg_k=3) if kind == "ksg_mi" else ndf.CorrelationMeasure(kind)
        g = ndf.ground_truth_field_device(f, meas, "v", "v", (0.0, 0.0, 0.0), (5, 4, 3), 11, 11)
        assert g.numel() == 0
    res = ndf.pair_estimators_device(f, "v", np.zeros(0, np.int64), np.zeros(0, np.int64), k=3)
    for v in (res.values() if isinstance(res, dict) else res):
        assert len(v) == 0
    torch.cuda.synchronize()


def test_ksg_extreme_sizes():
    """Size envelope of the GPU KSG: the smallest sample (M=2, k=1), the largest
    (M=4096 -- 224 KB of SMEM per pair, one CTA per SM -- with k=16), bit-exact counts
    and MI vs the oracle; past the envelope a ConfigError, not a fault."""
    rng = np.random.default_rng(21)
    for M, k, B in ((2, 1, 3), (3, 2, 3), (4096, 16, 3), (4096, 1, 2)):
        a = rng.standard_normal(M).astype(np.float32).astype(np.float64)
        b = np.stack([(0.6 * a + rng.standard_normal(M)).astype(np.float32).astype(np.float64)
                      for _ in range(B)])
        mi, counts = ndf.ksg_rows(a, b, k, return_counts=True)
        for s in range(B):
            assert mi[s] == O.ksg_mi(a, b[s], k), (M, k)
            if M <= 64:
                _, nx, ny = O.ksg_counts_bruteforce(a, b[s], k)
                assert np.array_equal(counts[s, 0], nx) and np.array_equal(counts[s, 1], ny)
    with pytest.raises(ndf.ConfigError):
        ndf.ksg_rows(np.zeros(4097), np.zeros((1, 4097)), 3)
    with pytest.raises(ndf.ConfigError):
        ndf.ksg_rows(np.arange(40.0), np.arange(40.0)[None], 17)
