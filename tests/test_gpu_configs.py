"""Every BASELINE config at its stated shape (VERDICT r1 "parity-test every config"):
full-size launches, checked against the oracle on seeded subsets.

* c1 / c2 NDF query over the full 250x352x20 grid (1.76 M vertices), fp32 / bf16 / fp16,
  both heads, parity (O(1) latent) and benched (1e-4 latent) models, vs the oracle on a
  seeded 2^16-vertex subset.
* c1 ground-truth Pearson GEMV at M = 1000 on the config-1 generator vs the oracle's
  pearson_against on a seeded vertex subset (<= 1e-5), reference vertex exactly 1.0.
* c2 KSG field at M = 1000 on the config-2 generator, bit-exact on a seeded subset.
* c4 bulk pairs: 4,096 pairs of config 4's list on its generator, KSG n_x / n_y counts
  bit-exact on every pair (scipy cKDTree, as the reference; brute force on 128 of them),
  MI bit-exact, Pearson <= 1e-12.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2307_02203_b200 as ndf  # noqa: E402
from oracle import ndf_oracle as O  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402

TOL = {"fp32": 1e-5, "bf16": 1e-2, "fp16": 1e-2}


def _om(model):
    return O.OracleModel(model.spec.fourier_octaves, model.grid_mu, model.grid_nu, model.weights,
                         model.biases, model.spec.merge, model.spec.activation,
                         model.spec.head_kind)


@pytest.mark.parametrize("cfg", [1, 2])
@pytest.mark.parametrize("grid_init", [1.0, 1e-4])
def test_full_grid_query_vs_oracle_subset(cfg, grid_init):
    w = W.CONFIGS[cfg]
    model = W.build_model(w, seed=0, grid_init=grid_init)
    ref = w.ref_position()
    idx = np.sort(np.random.default_rng(5).choice(w.n_vertices, 1 << 16, replace=False))
    want = O.reconstruct_field(_om(model), ref, w.dims, vertices=idx)
    for prec in ("fp32", "bf16", "fp16"):
        if prec == "fp32" and grid_init != 1.0:
            continue
        out = ndf.reconstruct_field_device(model.with_precision(prec), ref, ndf.ROLE_MU, w.dims)
        assert out.numel() == w.n_vertices
        err = float(np.max(np.abs(out.cpu().numpy()[idx] - want)))
        print(f"c{cfg} grid_init={grid_init:g} {prec}: max|err| {err:.3e} over 2^16 vertices")
        assert err <= TOL[prec], (cfg, grid_init, prec, err)


@pytest.fixture(scope="module")
def c1_ensemble():
    ens = W.generate_device(W.CONFIGS[1])
    yield ens
    del ens
    torch.cuda.empty_cache()


def test_c1_pearson_gemv_m1000_vs_oracle(c1_ensemble):
    w = W.CONFIGS[1]
    ref = w.ref_position()
    got = ndf.ground_truth_field_device(c1_ensemble, ndf.CorrelationMeasure("pearson"), "v", "v",
                                        ref, w.dims).cpu().numpy()
    assert got.shape == (w.n_vertices,)
    assert got[w.ref_flat()] == 1.0
    X = c1_ensemble.X.reshape(w.members, -1)
    idx = np.sort(np.random.default_rng(6).choice(w.n_vertices, 4096, replace=False))
    cols = X[:, torch.as_tensor(idx, device=X.device)].double().cpu().numpy().T   # (B, M)
    ref_vec = X[:, w.ref_flat()].double().cpu().numpy()
    # sample_many returns the stored values at grid nodes (ensemble.py:130-167, pinned
    # bitwise by tests/test_gpu_estimators.py::test_sample_many_bitwise)
    want = O.pearson_against(ref_vec, cols)
    want[np.isnan(want)] = 0.0
    want = want.astype(np.float32)
    err = float(np.max(np.abs(got[idx] - want)))
    print(f"c1 Pearson GEMV M=1000: max|err| {err:.3e} over 4096 vertices")
    assert err <= 1e-5


def test_c2_ksg_field_m1000_subset_bitexact():
    w = W.CONFIGS[2]
    ens = W.generate_device(w)
    ref = w.ref_position()
    got = ndf.ground_truth_field_device(ens, ndf.CorrelationMeasure("ksg_mi", ksg_k=8), "v", "v",
                                        ref, w.dims).cpu().numpy()
    X = ens.X.reshape(w.members, -1)
    idx = np.sort(np.random.default_rng(7).choice(w.n_vertices, 256, replace=False))
    cols = X[:, torch.as_tensor(idx, device=X.device)].double().cpu().numpy().T
    ref_vec = X[:, w.ref_flat()].double().cpu().numpy()
    want = np.array([O.ksg_mi(ref_vec, c, 8) for c in cols], dtype=np.float32)
    assert np.array_equal(got[idx], want)
    del ens
    torch.cuda.empty_cache()


def test_c4_pairs_counts_bitexact_4096():
    w = W.CONFIGS[4]
    ens = W.generate_device(w)
    pa, pb = W.pair_list(w, count=1 << 22, seed=2)
    sel = np.sort(np.random.default_rng(8).choice(pa.size, 4096, replace=False))
    pa, pb = pa[sel], pb[sel]
    res = ndf.pair_estimators_device(ens, "v", pa, pb, k=8, counts=True)
    cnt = res["ksg_counts"].cpu().numpy()
    mi = res["ksg_mi"].cpu().numpy()
    r = res["pearson"].cpu().numpy()
    X = ens.X.reshape(w.members, -1)
    A = X[:, torch.as_tensor(pa, device=X.device)].double().cpu().numpy().T
    B = X[:, torch.as_tensor(pb, device=X.device)].double().cpu().numpy().T
    assert np.max(np.abs(r - O.pearson_rowwise(A, B))) <= 1e-12
    for p in range(pa.size):
        _, n_x, n_y = O.ksg_counts_kdtree(A[p], B[p], 8)
        assert np.array_equal(cnt[p, 0], n_x) and np.array_equal(cnt[p, 1], n_y), p
        assert mi[p] == O.ksg_from_counts(n_x, n_y, 8), p
        if p < 128:
            _, bx, by = O.ksg_counts_bruteforce(A[p], B[p], 8)
            assert np.array_equal(bx, n_x) and np.array_equal(by, n_y), p
    del ens
    torch.cuda.empty_cache()
