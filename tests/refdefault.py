"""Shared helpers for the reference-default-family fixtures (tests/golden/ndf_refdefault.npz)."""

import numpy as np

import paper_2307_02203_b200 as ndf

SMALL = dict(levels=3, base_resolution=4, growth=2.0, log2_table_size=10, features_per_level=2,
             encoder_layers=2, decoder_layers=3, channels=16, fourier_octaves=4,
             activation="snake_alt", head="linear", precision="fp32")
CASES = {"mul": dict(merge="multiply"), "cat": dict(merge="concat"),
         "add2": dict(merge="add", var_mu="a", var_nu="b")}


def model_from_params(spec, params):
    """NdfModel from arrays in parameters() order (model.py:148-157)."""
    params = list(params)
    it = iter(params)
    grid_mu = next(it)
    grid_nu = grid_mu if spec.shared else next(it)

    def mlp(widths):
        ws, bs = [], []
        for _ in widths[:-1]:
            ws.append(next(it))
            bs.append(next(it))
        return ws, bs

    enc_mu = mlp(spec.encoder_widths())
    enc_nu = enc_mu if spec.shared else mlp(spec.encoder_widths())
    ws, bs = mlp(spec.decoder_widths())
    return ndf.NdfModel(spec, grid_mu, grid_nu, ws, bs, enc_mu, enc_nu)


def golden_case(g, name):
    spec = ndf.ModelSpec(**SMALL, **CASES[name])
    params = [g[f"{name}_param{i}"] for i in range(int(g[f"{name}_nparams"]))]
    return model_from_params(spec, params)


def oracle_model(model):
    """oracle/ndf_oracle.py restatement of an NdfModel (either family)."""
    from oracle import ndf_oracle as O
    spec = model.spec
    if spec.hash_grid:
        def grid(t):
            return O.HashGridSpec(t, tuple(spec.level_resolutions()), spec.log2_table_size)
        g_mu, g_nu = grid(model.grid_mu), grid(model.grid_nu)
    else:
        g_mu, g_nu = model.grid_mu, model.grid_nu
    return O.OracleModel(spec.fourier_octaves, g_mu, g_nu, model.weights, model.biases,
                         spec.merge, spec.activation, spec.head_kind,
                         tuple(model.enc_mu), tuple(model.enc_nu))
