"""Pin the CPU oracle against golden vectors produced by the unmodified reference.

These run without a GPU.  They establish that ``oracle/ndf_oracle.py`` (the
checker for every GPU parity test) reproduces the reference bit for bit on
every piece the reference can express.
"""

import numpy as np
import pytest

from oracle import ndf_oracle as O
import paper_2307_02203_b200 as ndf


def test_fourier_bitwise(golden):
    g = golden("encode")
    assert np.array_equal(O.fourier_encode(g["pos"], 6), g["fourier6"])


def test_fourier_known_answers():
    # reference tests/test_encoding.py:54-78
    out = O.fourier_encode(np.zeros((1, 3)), 3)[0]
    assert np.all(out[0::2] == 0.0) and np.all(out[1::2] == 1.0)
    out = O.fourier_encode(np.array([[0.5, 0.0, 0.0]]), 2)[0]
    assert out[0] == 1.0 and out[6] == np.sin(2 * np.pi * 0.5)


def test_dense_grid_matches_reference_hashgrid_bitwise(golden):
    g = golden("encode")
    r = int(g["dense_res"])
    table = g["dense_table"][0][: r ** 3].reshape(r, r, r, 16)
    assert np.array_equal(O.dense_grid_encode(g["pos"], table), g["dense_out"])


def test_dense_grid_vertex_exact():
    # reference tests/test_encoding.py:87-97 (vertex lookup exact), anisotropic
    rng = np.random.default_rng(0)
    table = rng.uniform(-1, 1, (3, 5, 7, 16)).astype(np.float32)
    for (i, j, k) in [(0, 0, 0), (6, 4, 2), (3, 1, 1)]:
        p = np.array([[2 * i / 6 - 1, 2 * j / 4 - 1, 2 * k / 2 - 1]])
        assert np.array_equal(O.dense_grid_encode(p, table)[0], table[k, j, i])


def test_mlp_bitwise(golden):
    g = golden("mlp")
    ws = [g[f"w{i}"] for i in range(4)]
    bs = [g[f"b{i}"] for i in range(4)]
    assert np.array_equal(O.mlp_forward(ws, bs, "snake_alt", g["x"]), g["y"])


@pytest.mark.parametrize("merge", ["add", "absdiff", "multiply"])
def test_reconstruct_reference_mode_bitwise(golden, merge):
    g = golden("ndf_refmode")
    grid = g[f"{merge}_grid"].reshape(4, 4, 4, 16)
    model = O.OracleModel(6, grid, grid, [g[f"{merge}_w{i}"] for i in range(4)],
                          [g[f"{merge}_b{i}"] for i in range(4)], merge, "snake_alt",
                          "linear")
    dims = tuple(int(d) for d in g["dims"])
    for r, ref in enumerate(g["refs"]):
        out = O.reconstruct_field(model, ref, dims)
        assert np.array_equal(out, g[f"{merge}_out{r}"])
        # batch invariance (reference tests/test_service.py:42-54)
        assert np.array_equal(O.reconstruct_field(model, ref, dims, batch_size=17), out)
    assert np.array_equal(model.forward(g[f"{merge}_p1"], g[f"{merge}_p2"]),
                          g[f"{merge}_fwd"])


def test_pearson_bitwise(golden):
    g = golden("pearson")
    got = O.pearson_rowwise(g["rw_a"], g["rw_b"])
    assert np.array_equal(np.isnan(got), np.isnan(g["rw_out"]))
    assert np.array_equal(got[~np.isnan(got)], g["rw_out"][~np.isnan(got)])
    assert got[3] == 1.0
    got = O.pearson_against(g["rw_a"][0], g["rw_b"])
    ok = ~np.isnan(g["against_out"])
    assert np.array_equal(got[ok], g["against_out"][ok])
    vals = [O.pearson(g["rw_a"][i], g["rw_b"][i]) for i in range(40) if i != 5]
    assert np.array_equal(np.array(vals), g["pearson_ab"])


def test_pearson_known_answers():
    # reference tests/test_measures.py:51-58
    assert O.pearson([1, 2, 3], [2, 4, 6]) == 1.0
    assert O.pearson([1, 2, 3], [3, 2, 1]) == -1.0
    assert O.pearson([1, 2, 3, 4], [1, 3, 2, 4]) == 0.8
    assert O.pearson([1.0, 1.0, 1.0], [1, 2, 3]) is None


def test_sample_many_bitwise(golden):
    g = golden("pearson")
    assert np.array_equal(O.sample_many(g["field"], g["sample_pos"]), g["sample_out"])


@pytest.mark.parametrize("name", ["node", "offnode"])
def test_ground_truth_pearson_bitwise(golden, name):
    g = golden("pearson")
    dims = tuple(int(d) for d in g[f"gt_{name}_dims"])
    out = O.ground_truth_field(g["field"], "pearson", g[f"gt_{name}_ref"], dims)
    assert np.array_equal(out, g[f"gt_{name}"])


def test_digamma_bitwise(golden):
    g = golden("ksg")
    assert np.array_equal(O.digamma(np.arange(1, 2001, dtype=np.float64)), g["psi"])


def test_ksg_kdtree_restatement_bitwise(golden):
    g = golden("ksg")
    for i in range(int(g["ksg_cases"])):
        a, b, k = g[f"ksg{i}_a"], g[f"ksg{i}_b"], int(g[f"ksg{i}_k"])
        assert O.ksg_mi(a, b, k) == float(g[f"ksg{i}_mi"]), i


def test_ksg_bruteforce_counts_equal_kdtree(golden):
    """The brute-force formulation (the GPU kernel's algorithm) reproduces the
    cKDTree counts exactly -- SURVEY 0.4 / H1."""
    g = golden("ksg")
    for i in range(int(g["ksg_cases"])):
        a, b, k = g[f"ksg{i}_a"], g[f"ksg{i}_b"], int(g[f"ksg{i}_k"])
        e1, x1, y1 = O.ksg_counts_bruteforce(a, b, k)
        e2, x2, y2 = O.ksg_counts_kdtree(a, b, k)
        assert np.array_equal(e1, e2) and np.array_equal(x1, x2) and np.array_equal(y1, y2)
        assert O.ksg_from_counts(x1, y1, k) == float(g[f"ksg{i}_mi"])


def test_ksg_bruteforce_many_seeds_m1000():
    # the BASELINE shape: M=1000, k=8, incl. fp32-quantised inputs with ties
    for s in range(6):
        r = np.random.default_rng(300 + s)
        x = r.standard_normal(1000).astype(np.float32).astype(np.float64)
        y = x + 0.5 * x ** 2 + 0.2 * np.sin(3 * x) + 0.3 * r.standard_normal(1000)
        if s == 0:
            y = np.round(y, 1)
        e1, x1, y1 = O.ksg_counts_bruteforce(x, y, 8)
        e2, x2, y2 = O.ksg_counts_kdtree(x, y, 8)
        assert np.array_equal(e1, e2) and np.array_equal(x1, x2) and np.array_equal(y1, y2)


def test_ground_truth_ksg_bitwise(golden):
    g = golden("ksg")
    dims = tuple(int(d) for d in g["gt_dims"])
    out = O.ground_truth_field(g["field"], "ksg_mi", g["gt_ref"], dims, k=int(g["gt_k"]))
    assert np.array_equal(out, g["gt_mi"])


@pytest.mark.parametrize("case", ["mul", "cat", "add2"])
def test_reference_family_restatement_bitwise(golden, case):
    """oracle HashGrid + encoder restatement == the unmodified reference, bit for bit."""
    import refdefault as R
    g = golden("ndf_refdefault")
    om = R.oracle_model(R.golden_case(g, case))
    dims = tuple(int(x) for x in g["dims"])
    for k, ref in enumerate(g["refs"]):
        assert np.array_equal(O.reconstruct_field(om, ref, dims), g[f"{case}_out{k}"])
    assert np.array_equal(O.reconstruct_field(om, g["refs"][0], dims, role="reference-is-nu"),
                          g[f"{case}_outnu"])
    assert np.array_equal(om.forward(g["p1"], g["p2"]), g[f"{case}_fwd"])


def test_reference_default_restatement_bitwise(golden):
    import refdefault as R
    g = golden("ndf_refdefault")
    m = ndf.NdfModel.build(ndf.ModelSpec.reference_default(), seed=0)
    om = R.oracle_model(m)
    dims = tuple(int(x) for x in g["dims"])
    assert np.array_equal(O.reconstruct_field(om, g["refs"][0], dims), g["default_out0"])
    assert np.array_equal(om.forward(g["p1"], g["p2"]), g["default_fwd"])


def test_activations_golden_bitwise(golden):
    """nn.py:23-32 (relu, snake, snake_alt) reproduced bit for bit on [-40, 40]."""
    g = golden("activations")
    for kind in ("relu", "snake", "snake_alt"):
        got = O.activation(kind, g["x"])
        assert got.dtype == np.float32
        assert np.array_equal(got, g[kind]), kind
