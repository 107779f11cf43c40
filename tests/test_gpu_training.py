"""Training-target drop-in on the GPU (training.py:111-119): off-grid position pairs,
samples kept in HBM, one Pearson / KSG launch per chunk -- vs the oracle's sample_many +
pearson_rowwise / ksg_mi on the same positions."""

import numpy as np
import pytest
import torch

import paper_2307_02203_b200 as ndf
from oracle import ndf_oracle as O
from paper_2307_02203_b200 import workloads as W

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


def test_targets_vs_oracle():
    w = W.CONFIGS[0]
    field = W.generate_host(w)
    grids = field.member_grids("v")
    rng = np.random.default_rng(7)
    p_mu = rng.uniform(-1.0, 1.0, (300, 3))
    p_nu = rng.uniform(-1.0, 1.0, (300, 3))
    p_nu[:20] = p_mu[:20]                     # identical pairs -> exactly 1.0
    p_nu[20:40] = O.grid_positions(w.dims)[rng.integers(0, w.n_vertices, 20)]   # nodes
    a = O.sample_many(grids, p_mu)
    b = O.sample_many(grids, p_nu)
    got = ndf.targets(field, ndf.CorrelationMeasure("pearson"), "v", "v", p_mu, p_nu)
    want = O.pearson_rowwise(a, b)
    assert got.dtype == np.float64 and got.shape == (300,)
    assert np.max(np.abs(got - want)) <= 1e-12
    assert np.all(got[:20] == 1.0)
    for k in (3, 8):
        got = ndf.targets(field, ndf.CorrelationMeasure("ksg_mi", ksg_k=k), "v", "v", p_mu, p_nu)
        want = np.array([O.ksg_mi(a[i], b[i], k) for i in range(len(a))])
        assert np.array_equal(got, want)
    # chunking does not change a bit
    from paper_2307_02203_b200.training import targets_device
    m = ndf.CorrelationMeasure("ksg_mi", ksg_k=3)
    whole = targets_device(field, m, "v", "v", p_mu, p_nu).cpu().numpy()
    chunked = targets_device(field, m, "v", "v", p_mu, p_nu, chunk=37).cpu().numpy()
    assert np.array_equal(whole, chunked)
    assert ndf.targets(field, m, "v", "v", np.zeros((0, 3)), np.zeros((0, 3))).shape == (0,)
    with pytest.raises(ndf.ParameterError):
        ndf.targets(field, m, "v", "v", p_mu, p_nu[:5])


def test_sample_pairs_with_targets_gpu():
    w = W.CONFIGS[0]
    field = W.generate_host(w)

    class Cfg:
        measure = ndf.CorrelationMeasure("ksg_mi", ksg_k=3)
        var_mu = var_nu = "v"

    p_mu, p_nu, t = ndf.sample_pairs_with_targets(field, Cfg, np.random.default_rng(3), 64,
                                                  on_grid=True)
    assert p_mu.shape == p_nu.shape == (64, 3) and np.all(np.isfinite(t))
    grids = field.member_grids("v")
    want = np.array([O.ksg_mi(x, y, 3) for x, y in zip(O.sample_many(grids, p_mu),
                                                       O.sample_many(grids, p_nu))])
    assert np.array_equal(t, want)


def test_compare_to_ground_truth_vs_oracle():
    """service.py:135-155 on the GPU: PSNR / max error / error field of the reconstruction
    against the ground-truth field, vs the same quantities from the oracle."""
    w = W.CONFIGS[0]
    field = W.generate_host(w)
    model = W.build_model(w, seed=0, grid_init=1.0)
    om = O.OracleModel(model.spec.fourier_octaves, model.grid_mu, model.grid_nu, model.weights,
                       model.biases, model.spec.merge, model.spec.activation, model.spec.head_kind)
    ref = w.ref_position()
    for role in (ndf.ROLE_MU, ndf.ROLE_NU):
        res = ndf.compare_to_ground_truth(model, field, ndf.CorrelationMeasure("pearson"), ref,
                                          w.dims, role)
        recon = O.reconstruct_field(om, ref, w.dims, role=role)
        truth = O.ground_truth_field(field.member_grids("v"), "pearson", ref, w.dims)
        truth = np.where(np.isnan(truth), 0.0, truth).astype(np.float32)
        err = recon.astype(np.float64) - truth.astype(np.float64)
        assert abs(res.psnr_db - ndf.psnr(recon, truth)) <= 1e-3
        assert abs(res.max_abs_err - np.max(np.abs(err))) <= 2e-5
        assert res.error_field.dims == w.dims
        assert np.max(np.abs(res.error_field.values - err.astype(np.float32))) <= 2e-5


def test_targets_two_variables_and_ksg_compare():
    """Targets across two variables (var_mu != var_nu, training.py:114-115) and the KSG
    ground truth in compare_to_ground_truth."""
    w = W.CONFIGS[0]
    f = W.generate_host(w)
    v = f.member_grids("v")
    u = np.ascontiguousarray(np.tanh(v) + 0.1 * v * v, dtype=np.float32)   # a second variable
    field = ndf.EnsembleField(f.domain, ("v", "u"), np.stack([v, u]))
    rng = np.random.default_rng(9)
    p_mu, p_nu = rng.uniform(-1, 1, (200, 3)), rng.uniform(-1, 1, (200, 3))
    for meas in (ndf.CorrelationMeasure("pearson"), ndf.CorrelationMeasure("ksg_mi", ksg_k=4)):
        got = ndf.targets(field, meas, "v", "u", p_mu, p_nu)
        a, b = O.sample_many(v, p_mu), O.sample_many(u, p_nu)
        if meas.kind == "pearson":
            assert np.max(np.abs(got - O.pearson_rowwise(a, b))) <= 1e-12
        else:
            assert np.array_equal(got, [O.ksg_mi(a[i], b[i], 4) for i in range(len(a))])
    model = W.build_model(w, seed=0, grid_init=1.0)
    res = ndf.compare_to_ground_truth(model, f, ndf.CorrelationMeasure("ksg_mi", ksg_k=3),
                                      w.ref_position(), w.dims)
    truth = O.ground_truth_field(v, "ksg_mi", w.ref_position(), w.dims, k=3)
    om = O.OracleModel(model.spec.fourier_octaves, model.grid_mu, model.grid_nu, model.weights,
                       model.biases, model.spec.merge, model.spec.activation, model.spec.head_kind)
    recon = O.reconstruct_field(om, w.ref_position(), w.dims)
    assert abs(res.psnr_db - ndf.psnr(recon, truth.astype(np.float32))) <= 1e-3


def test_sample_many_vertex_major_bitwise():
    """ndf_sample_many_vm (vertex-major source) == ndf_sample_many_ld, bit for bit, and the
    oracle's sample_many (ensemble.py:130-167)."""
    w = W.CONFIGS[0]
    field = W.generate_host(w)
    from paper_2307_02203_b200.ensemble import _device_view
    d = _device_view(field, "v")
    rng = np.random.default_rng(13)
    pos = np.concatenate([rng.uniform(-1.2, 1.2, (777, 3)), O.grid_positions(w.dims)[:50],
                          [[1.0, 1.0, 1.0], [-1.0, -1.0, -1.0]]])
    d.drop_derived()
    mm = d.sample_many(pos).cpu().numpy()
    d.vertex_major()
    vm = d.sample_many(pos).cpu().numpy()
    d.drop_derived()
    assert np.array_equal(mm, vm)
    assert np.array_equal(vm, O.sample_many(field.member_grids("v"), pos))
