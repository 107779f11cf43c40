"""GPU side of the drop-in boundary: the reference's own object structure (stand-ins
from tests/refobjects.py -- the reference package is not on the GPU box; the CPU test
tests/test_dropin.py ties the stand-ins to the real objects) goes straight into
reconstruct_field / forward / ground_truth_field, and NdfModel.embed / embed_nodes
(ndf_embed_points / ndf_embed_nodes) reproduce the oracle's embedding bit for bit
(model.py:169-177, pinned to the reference by tests/test_oracle.py)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2307_02203_b200 as ndf  # noqa: E402
import refobjects  # noqa: E402
from oracle import ndf_oracle as O  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402


def _models():
    w = W.CONFIGS[0]
    base = W.build_model(w, seed=0, grid_init=1.0)
    refd = ndf.NdfModel.build(ndf.ModelSpec.reference_default(var_mu="a", var_nu="b",
                                                              shared_encoder=False), seed=7)
    r = np.random.default_rng(3)
    for t in (refd.grid_mu, refd.grid_nu):
        t[:] = r.uniform(-1, 1, t.shape).astype(np.float32)
    return w, base, refd


def test_reference_structured_models_query_like_ours():
    w, base, refd = _models()
    ref = (0.137, -0.52, 0.91)
    # encoder-less dense model: the stand-in carries reference-layout (1, 2^T, C) tables
    spec_dense = ndf.ModelSpec(merge="add", fourier_octaves=6, levels=1, base_resolution=4,
                               log2_table_size=8, features_per_level=16, activation="snake_alt",
                               head="linear", channels=128)
    dense = ndf.NdfModel.build(spec_dense, seed=2)
    for ours in (dense, refd):
        stand_in = refobjects.ref_model_like(ours)
        got = ndf.reconstruct_field(stand_in, ref, ndf.ROLE_MU, w.dims).values
        want = ndf.reconstruct_field(ours, ref, ndf.ROLE_MU, w.dims).values
        assert np.array_equal(got, want)
        p1 = np.random.default_rng(1).uniform(-1, 1, (64, 3))
        p2 = np.random.default_rng(2).uniform(-1, 1, (64, 3))
        assert np.array_equal(ndf.forward(stand_in, p1, p2), ours.forward(p1, p2))
    # the converted model is cached per object; a training update is picked up
    stand_in = refobjects.ref_model_like(dense)
    a = ndf.reconstruct_field(stand_in, ref, ndf.ROLE_MU, w.dims).values
    stand_in.decoder.biases[-1][0] += 1.0
    b = ndf.reconstruct_field(stand_in, ref, ndf.ROLE_MU, w.dims).values
    assert np.allclose(b - a, 1.0, atol=1e-5)


def test_reference_structured_ensemble_ground_truth():
    w = W.CONFIGS[0]
    f = W.generate_host(w)
    stand_in = refobjects.RefEnsemble(*w.dims, f.values.copy())
    ref = w.ref_position()
    for meas in (ndf.CorrelationMeasure("pearson"), ndf.CorrelationMeasure("ksg_mi", ksg_k=3)):
        got = ndf.ground_truth_field(stand_in, meas, "v", "v", ref, w.dims).values
        want = ndf.ground_truth_field(f, meas, "v", "v", ref, w.dims).values
        assert np.array_equal(got, want)
    with pytest.raises(ndf.UnknownVariableError):
        ndf.ground_truth_field(stand_in, ndf.CorrelationMeasure("pearson"), "q", "q", ref, w.dims)


def test_embed_bitwise_vs_oracle():
    w, base, refd = _models()
    pts = np.concatenate([np.random.default_rng(4).uniform(-1.3, 1.3, (500, 3)),
                          O.grid_positions(w.dims)[:64], [[1.0, -1.0, 0.0]]])
    for model in (base, refd):
        for grid, table in ((model.grid_mu, model.grid_mu), ("nu", model.grid_nu)):
            om_table = table
            if model.spec.hash_grid:
                om_table = O.HashGridSpec(table, tuple(model.spec.level_resolutions()),
                                          model.spec.log2_table_size)
            got = model.embed(grid, pts)
            want = O.embed(pts, om_table, model.spec.fourier_octaves)
            assert got.dtype == np.float32 and got.shape == want.shape
            assert np.array_equal(got, want)
    # grid nodes, a vertex range of the config-1 grid (x fastest)
    w1 = W.CONFIGS[1]
    m1 = W.build_model(w1, seed=0, grid_init=1.0)
    v0, v1 = 123_456, 123_456 + 5000
    got = m1.embed_nodes("mu", w1.dims, v0, v1).cpu().numpy()
    want = O.embed(O.grid_positions_of(w1.dims, np.arange(v0, v1)), m1.grid_mu, 6)
    assert np.array_equal(got, want)
    # the reference family (HashGrid levels) over grid nodes: the generic per-point route
    dims = (9, 7, 3)
    hs = O.HashGridSpec(refd.grid_nu, tuple(refd.spec.level_resolutions()), refd.spec.log2_table_size)
    got = refd.embed_nodes("nu", dims).cpu().numpy()
    assert np.array_equal(got, O.embed(O.grid_positions(dims), hs, refd.spec.fourier_octaves))
    with pytest.raises(ndf.ParameterError):
        m1.embed(np.zeros_like(m1.grid_mu), pts)
    assert m1.embed("mu", np.zeros((0, 3))).shape == (0, 55)


def test_embed_nodes_row_segments_vs_oracle():
    """embed_rows_kernel (fp64 corners staged per row segment): bit-exact over whole grids,
    ragged ranges (odd starts: unaligned slabs), single-node axes and rows of several
    128-node segments."""
    from paper_2307_02203_b200.model import ModelSpec, NdfModel
    cases = [((32, 44, 4), (4, 6, 2), None),            # config 0, whole grid
             ((300, 5, 3), (75, 2, 2), (1, 1499)),      # 3 segments per row, odd ends
             ((1, 7, 5), (2, 2, 2), None),              # nx = 1
             ((130, 3, 1), (40, 2, 2), (127, 261)),     # latent finer along x than 1/4
             ((250, 352, 20), (63, 88, 5), (1_759_001, 1_760_000))]
    for dims, res, rng in cases:
        spec = ModelSpec(measure_kind="pearson", grid_resolution=res, precision="fp32", grid_init=1.0)
        m = NdfModel.build(spec, seed=3)
        V = dims[0] * dims[1] * dims[2]
        v0, v1 = rng if rng else (0, V)
        for branch, table in (("mu", m.grid_mu), ("nu", m.grid_nu)):
            got = m.embed_nodes(branch, dims, v0, v1).cpu().numpy()
            want = O.embed(O.grid_positions_of(dims, np.arange(v0, v1)), table, 6)
            assert np.array_equal(got, want), (dims, branch)


def test_swapped_roles_forward():
    """model.py:245-265: swapped.forward(p1, p2) == forward(p2, p1) -- bitwise for the
    commutative merges, to summation rounding for concat."""
    from paper_2307_02203_b200.model import ModelSpec, NdfModel
    rng = np.random.default_rng(8)
    p1, p2 = rng.uniform(-1, 1, (256, 3)), rng.uniform(-1, 1, (256, 3))
    for merge in ("sum_absdiff", "concat"):
        # separate branches (var_mu != var_nu): a shared concat model has no swapped twin
        # in the reference either (its decoder is not reordered, model.py:257)
        spec = ModelSpec(measure_kind="pearson", grid_resolution=(5, 6, 3), precision="fp32",
                         merge=merge, grid_init=1.0, var_mu="a", var_nu="b")
        m = NdfModel.build(spec, seed=2)
        got = m.swapped_roles().forward(p1, p2)
        want = m.forward(p2, p1)
        if merge == "concat":
            assert np.max(np.abs(got - want)) <= 1e-6
        else:
            assert np.array_equal(got, want)
