"""Generate golden vectors by running the UNMODIFIED reference package.

Run in the build container (the reference is importable only here):

    python tests/golden/make_golden.py

It imports ``ndf`` from ``/root/reference/pkg/src`` (read-only) and writes
small ``.npz`` fixtures next to this script.  The fixtures travel with the
repo; nothing at test time reads ``/root/reference``.

Fixtures (all inputs seeded, outputs produced by the reference itself):

* ``encode.npz``     fourier_encode (encoding.py:37-51) and a single dense
                     HashGrid level with F=16 (encoding.py:163-178) -- the
                     reference-expressible core of the BASELINE latent grid.
* ``mlp.npz``        Mlp.forward exact (nn.py:124-137), snake_alt.
* ``ndf_refmode.npz``reconstruct_field (service.py:46-84) of an
                     encoder-less, single-dense-level NdfModel with add /
                     absdiff / multiply merges (model.py:279-286): the
                     "reference mode" the GPU kernels must reproduce.
* ``ndf_refdefault.npz`` the reference's own architecture:
                     multi-level HashGrid with dense and hashed levels, encoder
                     MLPs, multiply / concat / add (two-branch) merges, SnakeAlt,
                     linear head -- parameters + reconstruct_field / forward
                     outputs; plus the default ModelSpec() built from seed 0
                     (parameter checksums and outputs).
* ``pearson.npz``    pearson / pearson_against / pearson_rowwise and
                     ground_truth_field(pearson) (measures.py:59-133, 273-295).
* ``activations.npz`` nn.activation (nn.py:23-32) -- relu, snake, snake_alt --
                     on seeded float32 inputs spanning [-40, 40]
                     (``python make_golden.py activations`` rewrites only this one).
* ``ksg.npz``        ksg_mi (measures.py:173-203) on seeded vectors incl.
                     duplicates and a constant vector, plus
                     ground_truth_field(ksg_mi) (measures.py:296-314), plus the
                     reference digamma on 1..2000 (measures.py:136-165).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"


def main():
    sys.path.insert(0, REF_SRC)
    import ndf
    from ndf.encoding import FourierConfig, HashGrid, HashGridConfig, fourier_encode
    from ndf.ensemble import EnsembleField, GridDomain, WhiteNoiseKernel, generate_synthetic
    from ndf.measures import (CorrelationMeasure, digamma, ground_truth_field, ksg_mi,
                              pearson, pearson_against, pearson_rowwise, sample_many)
    from ndf.model import ModelSpec, NdfModel
    from ndf.nn import Mlp
    from ndf.service import reconstruct_field

    assert ndf.__file__.startswith(REF_SRC), ndf.__file__

    # -- encoders ---------------------------------------------------------
    rng = np.random.default_rng(101)
    pos = np.concatenate([rng.uniform(-1.2, 1.2, (200, 3)),
                          np.array([[-1, -1, -1], [1, 1, 1], [0, 0, 0],
                                    [1 / 3, -1 / 3, 0.999999999999]])])
    four = fourier_encode(pos, FourierConfig(6))
    res = 5
    cfg = HashGridConfig(levels=1, base_resolution=res, log2_table_size=7,
                         features_per_level=16)
    tables = rng.uniform(-1, 1, (1, 128, 16)).astype(np.float32)
    grid = HashGrid(cfg, tables)
    genc = grid.encode(pos)
    np.savez_compressed(os.path.join(HERE, "encode.npz"), pos=pos, fourier6=four,
                        dense_res=res, dense_table=tables, dense_out=genc)

    # -- MLP ----------------------------------------------------------------
    mlp = Mlp.initialize([110, 128, 128, 128, 1], "snake_alt",
                         np.random.default_rng(5), np.float32)
    for b in mlp.biases:
        b[:] = np.random.default_rng(6).uniform(-0.5, 0.5, b.shape).astype(np.float32)
    x = np.random.default_rng(7).standard_normal((64, 110)).astype(np.float32)
    y = mlp.forward(x)
    arrays = {"x": x, "y": y}
    for i, (w, b) in enumerate(zip(mlp.weights, mlp.biases)):
        arrays[f"w{i}"] = w
        arrays[f"b{i}"] = b
    np.savez_compressed(os.path.join(HERE, "mlp.npz"), **arrays)

    # -- reference-mode NDF query ------------------------------------------
    arrays = {}
    dims = (9, 7, 5)
    refs = np.array([[0.3, -0.5, 0.2], [-1.0, 1.0, 0.0], [0.25, 0.5, 1.0]])
    arrays["dims"] = np.array(dims)
    arrays["refs"] = refs
    for merge in ("add", "absdiff", "multiply"):
        spec = ModelSpec(merge=merge, encoder_layers=0, levels=1, base_resolution=4,
                         log2_table_size=6, features_per_level=16, fourier_octaves=6,
                         decoder_layers=4, channels=128)
        model = NdfModel.build(spec, seed=3)
        # O(1) grid values so gather errors are not hidden (SURVEY 8.0 "Grid init")
        model.grid_mu.tables[:] = np.random.default_rng(8).uniform(
            -1, 1, model.grid_mu.tables.shape).astype(np.float32)
        for b in model.decoder.biases:
            b[:] = np.random.default_rng(9).uniform(-0.2, 0.2, b.shape).astype(np.float32)
        arrays[f"{merge}_grid"] = model.grid_mu.tables[0].copy()
        for i, (w, b) in enumerate(zip(model.decoder.weights, model.decoder.biases)):
            arrays[f"{merge}_w{i}"] = w
            arrays[f"{merge}_b{i}"] = b
        for r, ref in enumerate(refs):
            arrays[f"{merge}_out{r}"] = reconstruct_field(model, ref, "reference-is-mu",
                                                         dims).values
        p1 = np.random.default_rng(10).uniform(-1, 1, (50, 3))
        p2 = np.random.default_rng(11).uniform(-1, 1, (50, 3))
        arrays[f"{merge}_p1"] = p1
        arrays[f"{merge}_p2"] = p2
        arrays[f"{merge}_fwd"] = model.forward(p1, p2)
    np.savez_compressed(os.path.join(HERE, "ndf_refmode.npz"), **arrays)

    # -- reference default family: HashGrid + encoder MLPs -------------
    arrays = {}
    dims = (9, 7, 5)
    arrays["dims"] = np.array(dims)
    arrays["refs"] = refs
    p1 = np.random.default_rng(20).uniform(-1.05, 1.05, (40, 3))
    p2 = np.random.default_rng(21).uniform(-1.05, 1.05, (40, 3))
    arrays["p1"], arrays["p2"] = p1, p2
    small = dict(levels=3, base_resolution=4, growth=2.0, log2_table_size=10,
                 features_per_level=2, encoder_layers=2, decoder_layers=3, channels=16,
                 fourier_octaves=4)      # res 4, 8 dense; 16^3 > 2^10 hashed
    cases = [("mul", dict(merge="multiply")), ("cat", dict(merge="concat")),
             ("add2", dict(merge="add", var_mu="a", var_nu="b"))]
    for name, extra in cases:
        spec = ModelSpec(**small, **extra)
        model = NdfModel.build(spec, seed=31)
        r = np.random.default_rng(32)
        grids = [model.grid_mu] if spec.shared else [model.grid_mu, model.grid_nu]
        for g in grids:          # O(1) tables so the hash gather is not hidden
            g.tables[:] = r.uniform(-1, 1, g.tables.shape).astype(np.float32)
        mlps = [model.enc_mu, model.decoder] if spec.shared else \
            [model.enc_mu, model.enc_nu, model.decoder]
        for mlp in mlps:
            for b in mlp.biases:
                b[:] = r.uniform(-0.2, 0.2, b.shape).astype(np.float32)
        for i, prm in enumerate(model.parameters()):
            arrays[f"{name}_param{i}"] = prm
        arrays[f"{name}_nparams"] = np.array(len(model.parameters()))
        for k, ref in enumerate(refs):
            arrays[f"{name}_out{k}"] = reconstruct_field(model, ref, "reference-is-mu", dims).values
        arrays[f"{name}_outnu"] = reconstruct_field(model, refs[0], "reference-is-nu", dims).values
        arrays[f"{name}_fwd"] = model.forward(p1, p2)
    # the unmodified default ModelSpec(): parameters regenerated from the seed (checked
    # through per-array sums), outputs of the reference itself
    model = NdfModel.build(ModelSpec(), seed=0)
    arrays["default_param_sums"] = np.array([float(np.sum(p, dtype=np.float64))
                                             for p in model.parameters()])
    arrays["default_param_first"] = np.array([float(p.ravel()[0]) for p in model.parameters()])
    for k, ref in enumerate(refs):
        arrays[f"default_out{k}"] = reconstruct_field(model, ref, "reference-is-mu", dims).values
    arrays["default_fwd"] = model.forward(p1, p2)
    np.savez_compressed(os.path.join(HERE, "ndf_refdefault.npz"), **arrays)

    # -- Pearson --------------------------------------------------------------
    arrays = {}
    rng = np.random.default_rng(12)
    a = rng.standard_normal((40, 33))
    b = rng.standard_normal((40, 33)) + 0.5 * a
    b[3] = a[3]            # exact self row -> 1.0
    b[5] = 2.0             # degenerate -> NaN
    arrays["rw_a"], arrays["rw_b"] = a, b
    arrays["rw_out"] = pearson_rowwise(a, b)
    arrays["against_out"] = pearson_against(a[0], b)
    arrays["pearson_ab"] = np.array([pearson(a[i], b[i]) for i in range(40) if i != 5])
    field = generate_synthetic(GridDomain(6, 5, 4), 64, ("v",), WhiteNoiseKernel(), seed=13)
    vals = field.values.copy()
    vals[0, :, 3, 2, 1] = 0.25     # one constant (degenerate) node
    field = EnsembleField(field.domain, field.variables, vals)
    arrays["field"] = field.values[0]
    for name, ref, gdims in (("node", (-1.0, 0.5, 1 / 3), (6, 5, 4)),
                             ("offnode", (0.1, -0.3, 0.7), (7, 4, 3))):
        gt = ground_truth_field(field, CorrelationMeasure("pearson"), "v", "v", ref, gdims)
        arrays[f"gt_{name}_ref"] = np.array(ref)
        arrays[f"gt_{name}_dims"] = np.array(gdims)
        arrays[f"gt_{name}"] = gt.values
    qpos = np.random.default_rng(14).uniform(-1, 1, (20, 3))
    arrays["sample_pos"] = qpos
    arrays["sample_out"] = sample_many(field, "v", qpos)
    np.savez_compressed(os.path.join(HERE, "pearson.npz"), **arrays)

    # -- KSG -------------------------------------------------------------------
    arrays = {}
    cases = []
    for s in range(12):
        r = np.random.default_rng(200 + s)
        n = int(r.integers(20, 400))
        x = r.standard_normal(n)
        y = 0.6 * x + 0.8 * r.standard_normal(n)
        if s % 4 == 1:
            x = np.round(x, 1)
            y = np.round(y, 1)
        if s % 4 == 2:
            y = x + 0.5 * x ** 2 + 0.2 * np.sin(3 * x)
        if s == 3:
            x = np.zeros(n)
        if s % 4 == 3 and s != 3:
            x = x.astype(np.float32).astype(np.float64)
        k = int(r.integers(1, 9))
        cases.append((x, y, k))
    for i, (x, y, k) in enumerate(cases):
        arrays[f"ksg{i}_a"], arrays[f"ksg{i}_b"] = x, y
        arrays[f"ksg{i}_k"] = np.array(k)
        arrays[f"ksg{i}_mi"] = np.array(ksg_mi(x, y, k))
    arrays["ksg_cases"] = np.array(len(cases))
    f2 = generate_synthetic(GridDomain(4, 3, 3), 60, ("v",), WhiteNoiseKernel(), seed=15)
    arrays["field"] = f2.values[0]
    gt = ground_truth_field(f2, CorrelationMeasure("ksg_mi", ksg_k=4), "v", "v",
                            (1.0, -1.0, 0.0), (4, 3, 3))
    arrays["gt_ref"] = np.array((1.0, -1.0, 0.0))
    arrays["gt_dims"] = np.array((4, 3, 3))
    arrays["gt_k"] = np.array(4)
    arrays["gt_mi"] = gt.values
    arrays["psi"] = digamma(np.arange(1, 2001, dtype=np.float64))
    np.savez_compressed(os.path.join(HERE, "ksg.npz"), **arrays)
    print("golden fixtures written to", HERE)


def activations():
    sys.path.insert(0, REF_SRC)
    import ndf
    from ndf.nn import activation
    assert ndf.__file__.startswith(REF_SRC), ndf.__file__
    rng = np.random.default_rng(11)
    x = np.concatenate([rng.standard_normal(4096) * 3.0, rng.uniform(-40, 40, 4096),
                        [0.0, -0.0, 1e-30, -1e-30, 40.0, -40.0]]).astype(np.float32)
    arrays = {"x": x}
    for kind in ("relu", "snake", "snake_alt"):
        arrays[kind] = activation(kind, x)
    np.savez_compressed(os.path.join(HERE, "activations.npz"), **arrays)
    print("activations.npz written to", HERE)


if __name__ == "__main__":
    if sys.argv[1:] == ["activations"]:
        activations()
    else:
        main()
        activations()
