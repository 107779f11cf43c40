"""GPU tests of the batched workloads: multi-reference cube (config 3), bulk estimator
pairs (config 4) and the single-rank NCCL path of the sharded query."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2307_02203_b200 as ndf  # noqa: E402
from oracle import ndf_oracle as O  # noqa: E402
from paper_2307_02203_b200 import workloads as W  # noqa: E402


@pytest.mark.parametrize("precision", ["fp16", "bf16"])
@pytest.mark.parametrize("merge", ["sum_absdiff", "add"])
def test_multi_reference_cube_equals_single_queries(precision, merge):
    """The cube row of a reference is its single query rounded to fp16, bit for bit:
    sum_absdiff runs both on the ping-pong kernel (per-reference tables), the other
    merges both on the classic schedule (query embedding reused across references)."""
    from dataclasses import replace
    dims = (70, 40, 6)
    spec = ndf.ModelSpec.baseline(dims, 4, precision=precision, grid_init=1.0)
    if merge != "sum_absdiff":
        spec = replace(spec, merge=merge)
    model = ndf.NdfModel.build(spec, seed=3)
    rng = np.random.default_rng(0)
    refs = np.concatenate([rng.uniform(-1, 1, (5, 3)), [[-1.0, 1.0, 0.2]]])
    V = int(np.prod(dims))
    cube = ndf.reconstruct_multi_device(model, refs, ndf.ROLE_MU, dims).cpu()
    assert cube.shape == (len(refs), V) and cube.dtype == torch.float16
    for r, ref in enumerate(refs):
        single = ndf.reconstruct_field_device(model, ref, ndf.ROLE_MU, dims).cpu()
        assert torch.equal(cube[r], single.half()), (merge, r)
    # vertex sub-range into a strided output
    out = torch.zeros((len(refs), 2000), dtype=torch.float16, device="cuda")
    ndf.reconstruct_multi_device(model, refs, ndf.ROLE_MU, dims, 1000, 2500, out=out)
    assert torch.equal(out[:, :1500].cpu(), cube[:, 1000:2500])
    # a one-reference cube through the multi-reference entry point
    one = ndf.reconstruct_multi_device(model, refs[2:3], ndf.ROLE_MU, dims).cpu()
    assert torch.equal(one[0], cube[2])


def test_multi_reference_oracle_spot_check():
    w = W.CONFIGS[0]
    model = W.build_model(w, seed=0, grid_init=1.0).with_precision("fp16")
    refs = np.array([w.ref_position(), (0.5, -0.5, 1.0), (-1.0, -1.0, -1.0)])
    cube = ndf.reconstruct_multi_device(model, refs, ndf.ROLE_MU, w.dims).float().cpu().numpy()
    om = O.OracleModel(6, model.grid_mu, model.grid_nu, model.weights, model.biases,
                       model.spec.merge, model.spec.activation, model.spec.head_kind)
    for r, ref in enumerate(refs):
        want = O.reconstruct_field(om, ref, w.dims)
        assert np.max(np.abs(cube[r] - want)) <= 1e-2


def test_bulk_pairs_vs_oracle():
    w = W.Workload("c4_small", (30, 24, 4), 400, (8, 8, 2), 4, "fp16", "ksg_mi", nonlinear=True,
                   ref_vertex=(15, 12, 2), seed=2311)
    ens = W.generate_device(w)
    pa, pb = W.pair_list(w, count=300, seed=2)
    pa[0] = pb[0]
    res = ndf.pair_estimators_device(ens, "v", pa, pb, k=8)
    X = ens.X.reshape(w.members, -1).cpu().numpy()
    r = res["pearson"].cpu().numpy()
    mi = res["ksg_mi"].cpu().numpy()
    want_r = O.pearson_rowwise(X[:, pa].T, X[:, pb].T)
    assert r[0] == 1.0
    assert np.max(np.abs(r - want_r)) <= 1e-12
    for p in range(0, 300, 11):
        assert mi[p] == O.ksg_mi(X[:, pa[p]].astype(np.float64), X[:, pb[p]].astype(np.float64), 8)
    with pytest.raises(ndf.ParameterError):
        ndf.pair_estimators_device(ens, "v", [0], [w.n_vertices], k=8)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sharded_paths_single_rank_nccl():
    """The four sharded paths through NCCL on one rank (the gloo world-2 tests cover the
    bookkeeping; one GPU is all this run has): each equals its unsharded call bitwise,
    the ground-truth field through the V-slice window + reference broadcast."""
    import torch.distributed as dist
    from paper_2307_02203_b200 import parallel as P
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        w = W.CONFIGS[0]
        ref = w.ref_position()
        for prec in ("bf16", "fp16"):
            model = W.build_model(w, seed=0, grid_init=1.0).with_precision(prec)
            got = P.reconstruct_field_sharded(model, ref, ndf.ROLE_MU, w.dims)
            assert torch.equal(got, ndf.reconstruct_field_device(model, ref, ndf.ROLE_MU, w.dims))
            refs = np.array([ref, (0.3, -0.2, 0.9), (-1.0, 1.0, 0.0)])
            cube = P.reconstruct_multi_sharded(model, refs, ndf.ROLE_MU, w.dims)
            assert torch.equal(cube, ndf.reconstruct_multi_device(model, refs, ndf.ROLE_MU, w.dims))
        f = W.generate_host(w)
        for meas in (ndf.CorrelationMeasure("pearson"), ndf.CorrelationMeasure("ksg_mi", ksg_k=4)):
            for r in (ref, (0.123, -0.45, 0.77)):          # node and off-node references
                got = P.ground_truth_field_sharded(f, meas, "v", "v", r, w.dims)
                want = ndf.ground_truth_field_device(f, meas, "v", "v", r, w.dims)
                assert torch.equal(got.nan_to_num(), want.nan_to_num()), (meas.kind, r)
        pa, pb = W.pair_list(w, count=500, seed=2)
        got = P.pair_estimators_sharded(f, "v", pa, pb, k=4)
        want = ndf.pair_estimators_device(f, "v", pa, pb, k=4)
        for name in ("pearson", "ksg_mi"):
            assert torch.equal(got[name].nan_to_num(), want[name].nan_to_num()), name
    finally:
        dist.destroy_process_group()


def test_column_window_matches_whole_variable():
    """DeviceEnsemble.window (a rank's V-slice): Pearson / KSG over vertices of the
    window equal the whole-variable results bitwise; sampling inside the window too."""
    w = W.CONFIGS[0]
    f = W.generate_host(w)
    X = f.member_grids("v")
    c0, c1 = 1000, 3900
    win = ndf.DeviceEnsemble.window(X, c0, c1)
    full = ndf.DeviceEnsemble.from_numpy(X)
    ref = w.ref_position()
    vec = full.sample_many(np.asarray(ref).reshape(1, 3))[0]
    for meas in (ndf.CorrelationMeasure("pearson"), ndf.CorrelationMeasure("ksg_mi", ksg_k=3)):
        got = ndf.ground_truth_field_device(win, meas, "v", "v", ref, w.dims, 1200, 3000, ref_vec=vec)
        want = ndf.ground_truth_field_device(full, meas, "v", "v", ref, w.dims, 1200, 3000)
        assert torch.equal(got, want), meas.kind
    pos = ndf.grid_positions(w.dims)[[1500, 2222]] + 1e-3
    assert torch.equal(win.sample_many(pos), full.sample_many(pos))
    with pytest.raises(ndf.ParameterError):
        ndf.ground_truth_field_device(win, ndf.CorrelationMeasure("pearson"), "v", "v", ref,
                                      w.dims, 500, 3000, ref_vec=vec)
    with pytest.raises(ndf.ParameterError):
        win.zscore()


def test_load_ensemble_device_streams_one_variable(tmp_path):
    """an NDFE variable streamed through pinned double buffers into HBM
    equals load_ensemble's bytes; truncation / unknown variables / non-finite values
    raise the reference's errors."""
    rng = np.random.default_rng(11)
    vals = rng.standard_normal((3, 37, 5, 9, 13)).astype(np.float32)
    f = ndf.EnsembleField(ndf.GridDomain(13, 9, 5), ("a", "b", "c"), vals)
    p = tmp_path / "e.ndfe"
    ndf.save_ensemble(f, p)
    host = ndf.load_ensemble(p)
    for var in ("a", "b", "c"):
        dev = ndf.load_ensemble_device(p, var, chunk_bytes=1 << 20)   # several chunks
        assert torch.equal(dev.X.cpu(), torch.from_numpy(np.array(host.member_grids(var))))
    big = rng.standard_normal((1, 300, 20, 30, 40)).astype(np.float32)   # 28.8 MB > 1 MiB chunks
    g = ndf.EnsembleField(ndf.GridDomain(40, 30, 20), ("v",), big)
    q = tmp_path / "big.ndfe"
    ndf.save_ensemble(g, q)
    assert torch.equal(ndf.load_ensemble_device(q, "v", chunk_bytes=1 << 20).X.cpu(),
                       torch.from_numpy(big[0]))
    with pytest.raises(ndf.UnknownVariableError):
        ndf.load_ensemble_device(p, "zz")
    trunc = tmp_path / "t.ndfe"
    trunc.write_bytes(p.read_bytes()[:-4])
    with pytest.raises(ndf.CorruptFileError):
        ndf.load_ensemble_device(trunc, "a")
    raw = bytearray(p.read_bytes())       # one NaN inside variable "b" (EnsembleField
    off = len(raw) - vals.nbytes + vals[0].nbytes + 7 * 4   # itself rejects non-finite)
    raw[off:off + 4] = np.array([np.nan], dtype="<f4").tobytes()
    r = tmp_path / "nan.ndfe"
    r.write_bytes(bytes(raw))
    ndf.load_ensemble_device(r, "a")      # the other variables stay loadable
    with pytest.raises(ndf.DataError):
        ndf.load_ensemble_device(r, "b")
