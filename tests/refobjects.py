"""Stand-ins with the attribute structure of the reference's own objects, for GPU tests
(the reference package is not on the GPU box): ``ndf.model.NdfModel`` (spec, HashGrid
grids with ``.tables``, ``Mlp`` encoders / decoder with ``weights``, ``biases``, ``act``,
``parameters()``; model.py:105-157, nn.py:40-110) and ``ndf.ensemble.EnsembleField``
(``domain``, ``variables``, ``member_grids``; ensemble.py:65-112).  The CPU test
tests/test_dropin.py checks the same conversion on the unmodified reference objects."""

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class RefSpec:                  # the reference ModelSpec's fields (model.py:29-46)
    var_mu: str = "v"
    var_nu: str = "v"
    measure_kind: str = "pearson"
    merge: str = "multiply"
    shared_encoder: bool = None
    fourier_octaves: int = 4
    levels: int = 6
    base_resolution: int = 16
    growth: float = 2.0
    log2_table_size: int = 16
    features_per_level: int = 2
    encoder_layers: int = 4
    decoder_layers: int = 4
    channels: int = 32

    @property
    def shared(self):
        return self.var_mu == self.var_nu if self.shared_encoder is None else self.shared_encoder


class RefGrid:
    def __init__(self, tables):
        self.tables = tables


class RefMlp:
    def __init__(self, weights, biases, act="snake_alt"):
        self.weights, self.biases, self.act = weights, biases, act

    def parameters(self):
        out = []
        for w, b in zip(self.weights, self.biases):
            out.extend((w, b))
        return out


class RefModel:
    def __init__(self, spec, grid_mu, grid_nu, enc_mu, enc_nu, decoder):
        self.spec, self.grid_mu, self.grid_nu = spec, grid_mu, grid_nu
        self.enc_mu, self.enc_nu, self.decoder = enc_mu, enc_nu, decoder

    def parameters(self):
        p = [self.grid_mu.tables]
        if not self.spec.shared:
            p.append(self.grid_nu.tables)
        p += self.enc_mu.parameters()
        if not self.spec.shared:
            p += self.enc_nu.parameters()
        return p + self.decoder.parameters()


def ref_model_like(model):
    """A reference-structured object holding (copies of) ``model``'s parameters, with
    the tables in the reference's (levels, 2^T, F) layout."""
    s = model.spec
    spec = RefSpec(var_mu=s.var_mu, var_nu=s.var_nu, measure_kind=s.measure_kind, merge=s.merge,
                   shared_encoder=s.shared_encoder, fourier_octaves=s.fourier_octaves,
                   levels=s.levels, base_resolution=s.base_resolution, growth=s.growth,
                   log2_table_size=s.log2_table_size, features_per_level=s.features_per_level,
                   encoder_layers=s.encoder_layers, decoder_layers=s.decoder_layers,
                   channels=s.channels)

    def tables(g):
        if s.hash_grid:
            return g.copy()
        T = 1 << s.log2_table_size
        t = np.zeros((1, T, s.features_per_level), np.float32)
        flat = g.reshape(-1, s.features_per_level)
        t[0, :flat.shape[0]] = flat
        return t
    gm = RefGrid(tables(model.grid_mu))
    gn = gm if s.shared else RefGrid(tables(model.grid_nu))
    em = RefMlp([w.copy() for w in model.enc_mu[0]], [b.copy() for b in model.enc_mu[1]],
                s.activation)
    en = em if s.shared else RefMlp([w.copy() for w in model.enc_nu[0]],
                                    [b.copy() for b in model.enc_nu[1]], s.activation)
    dec = RefMlp([w.copy() for w in model.weights], [b.copy() for b in model.biases], s.activation)
    return RefModel(spec, gm, gn, em, en, dec)


@dataclass(frozen=True)
class RefDomain:
    nx: int
    ny: int
    nz: int


class RefEnsemble:
    def __init__(self, nx, ny, nz, values, variables=("v",)):
        self.domain = RefDomain(nx, ny, nz)
        self.variables = tuple(variables)
        self.values = values

    def member_grids(self, name):
        return self.values[self.variables.index(name)]
