"""NDF model: spec, parameters, GPU-resident state, NDFM IO (drop-in for model.py).

``ModelSpec`` keeps every field of the reference (``model.py:29-102``) and
adds the BASELINE.json architecture knobs: a dense
anisotropic latent grid (``grid_resolution``), the ``sum_absdiff`` merge,
SiLU hidden activations, a tanh/softplus ``head`` and the query
``precision`` ("fp32" = exact SIMT kernel, "bf16" = tcgen05 kernel).

Two model families share the GPU path:

* dense: one dense latent level per branch, no encoder MLP -- BASELINE's
  architecture (anisotropic ``grid_resolution``) and the reference's
  ``encoder_layers=0`` single-dense-level ablation; every precision;
* reference: the reference's own architecture -- multi-level
  HashGrid tables ``(levels, 2^T, F)`` (encoding.py:120-178), per-branch
  encoder MLPs (model.py:131-142) and any merge -- on the exact fp32 kernel.
  ``ModelSpec.reference_default()`` is the reference ModelSpec() default
  (SnakeAlt, linear head), and reference NDFM files load unchanged.
"""

from __future__ import annotations

import json
import struct
from dataclasses import asdict, dataclass, replace

import numpy as np

from . import _native as N
from .errors import ConfigError, FormatError, ModelCorruptError, ParameterError, ShapeError

NDFM_MAGIC = b"NDFM"
NDFM_VERSION = 1

MERGE_MODES = ("multiply", "concat", "add", "absdiff", "sum_absdiff")
ACTIVATIONS = ("relu", "snake", "snake_alt", "silu")
HEADS = ("linear", "tanh", "softplus")
PRECISIONS = ("fp32", "bf16", "fp16")


@dataclass(frozen=True)
class ModelSpec:
    """Architecture descriptor (model.py:29-102 + BASELINE extensions)."""

    var_mu: str = "v"
    var_nu: str = "v"
    measure_kind: str = "pearson"
    merge: str = "sum_absdiff"
    shared_encoder: bool | None = None
    fourier_octaves: int = 6
    levels: int = 1
    base_resolution: int = 16
    growth: float = 2.0
    log2_table_size: int = 16
    features_per_level: int = 16
    encoder_layers: int = 0
    decoder_layers: int = 4
    channels: int = 128
    # --- BASELINE extensions (precision: "fp32" exact SIMT, "bf16"/"fp16" tcgen05) ---
    grid_resolution: tuple | None = None     # dense latent (rx, ry, rz); None = isotropic level 0
    activation: str = "silu"
    head: str | None = None                  # None: tanh for pearson, softplus for ksg_mi
    precision: str = "fp32"
    grid_init: float = 1e-4                  # U(-s, s) latent init (encoding.py:139-147)

    def __post_init__(self):
        if self.merge not in MERGE_MODES:
            raise ConfigError(f"merge must be one of {MERGE_MODES}, got {self.merge!r}")
        if self.encoder_layers < 0 or self.decoder_layers < 1:
            raise ConfigError("need encoder_layers >= 0 and decoder_layers >= 1")
        if self.channels < 1:
            raise ConfigError("channels must be >= 1")
        if self.shared and self.var_mu != self.var_nu:
            raise ConfigError("shared encoders require a self-correlation pair")
        if self.measure_kind not in ("pearson", "ksg_mi"):
            raise ConfigError(f"unknown measure kind {self.measure_kind!r}")
        if self.activation not in ACTIVATIONS:
            raise ConfigError(f"activation must be one of {ACTIVATIONS}")
        if self.head is not None and self.head not in HEADS:
            raise ConfigError(f"head must be one of {HEADS}")
        if self.precision not in PRECISIONS:
            raise ConfigError(f"precision must be one of {PRECISIONS}")
        if self.grid_resolution is not None:
            gr = tuple(int(r) for r in self.grid_resolution)
            if len(gr) != 3 or min(gr) < 2:
                raise ConfigError("grid_resolution needs three axes with >= 2 nodes")
            object.__setattr__(self, "grid_resolution", gr)
        if self.fourier_octaves < 0:
            raise ConfigError("fourier_octaves must be >= 0")

    @property
    def shared(self) -> bool:
        if self.shared_encoder is None:
            return self.var_mu == self.var_nu
        return self.shared_encoder

    @property
    def head_kind(self) -> str:
        if self.head is not None:
            return self.head
        return "tanh" if self.measure_kind == "pearson" else "softplus"

    @property
    def hash_grid(self) -> bool:
        """True for the reference family: HashGrid tables and/or encoder MLPs."""
        if self.grid_resolution is not None:
            return False
        r0 = int(round(self.base_resolution))
        return (self.levels > 1 or self.encoder_layers > 0
                or r0 ** 3 > (1 << self.log2_table_size))

    def level_resolutions(self) -> list:
        """Per-level lattice resolution (encoding.py:82-83)."""
        return [int(round(self.base_resolution * self.growth ** lv)) for lv in range(self.levels)]

    def encoder_widths(self) -> list:
        return [self.embed_dim] + [self.channels] * self.encoder_layers

    @property
    def latent_resolution(self) -> tuple:
        if self.grid_resolution is not None:
            return self.grid_resolution
        r = int(round(self.base_resolution))
        return (r, r, r)

    @property
    def embed_dim(self) -> int:
        return 3 + 6 * self.fourier_octaves + self.levels * self.features_per_level

    @property
    def encoder_output_dim(self) -> int:
        return self.channels if self.encoder_layers else self.embed_dim

    @property
    def decoder_input_dim(self) -> int:
        base = self.encoder_output_dim
        return 2 * base if self.merge in ("concat", "sum_absdiff") else base

    def decoder_widths(self) -> list:
        return [self.decoder_input_dim] + [self.channels] * (self.decoder_layers - 1) + [1]

    def check_gpu_supported(self) -> None:
        """Raise ConfigError if the spec is outside the GPU kernels' envelope."""
        if self.hash_grid:
            if self.precision != "fp32":
                raise ConfigError("HashGrid / encoder models run on the exact fp32 path "
                                  "(precision='fp32'); the tcgen05 kernel needs the dense grid")
            if self.levels > N.NDF_MAX_LEVELS or self.levels * self.features_per_level > 64:
                raise ConfigError("HashGrid exceeds the kernel envelope (<= 16 levels, "
                                  "levels x features <= 64)")
            if not 1 <= self.log2_table_size < 31:
                raise ConfigError("log2_table_size must be in [1, 31)")
            if min(self.level_resolutions()) < 2:
                raise ConfigError("level resolution must be >= 2")
            ew = self.encoder_widths()
            if len(ew) - 1 > N.NDF_MAX_LAYERS or max(ew) > N.NDF_MAX_WIDTH:
                raise ConfigError("encoder exceeds the kernel envelope (<= 8 layers, width <= 256)")
        widths = self.decoder_widths()
        if len(widths) - 1 > N.NDF_MAX_LAYERS or max(widths) > N.NDF_MAX_WIDTH:
            raise ConfigError("decoder exceeds the kernel envelope (<= 8 layers, width <= 256)")
        if self.fourier_octaves > 12 or self.features_per_level > 64:
            raise ConfigError("encoder exceeds the kernel envelope (L <= 12, C <= 64)")

    @classmethod
    def reference_default(cls, **kw) -> "ModelSpec":
        """The reference's ModelSpec() default (model.py:29-46): 6-level HashGrid,
        4-layer SnakeAlt encoders and decoder, 32 channels, multiply merge, linear head."""
        fields = dict(merge="multiply", fourier_octaves=4, levels=6, base_resolution=16,
                      growth=2.0, log2_table_size=16, features_per_level=2, encoder_layers=4,
                      decoder_layers=4, channels=32, activation="snake_alt", head="linear",
                      precision="fp32")
        fields.update(kw)
        return cls(**fields)

    @classmethod
    def baseline(cls, dims, factor: int, measure_kind: str = "pearson",
                 precision: str = "fp32", **kw) -> "ModelSpec":
        """BASELINE.json model: 16-ch latent at 1/factor resolution, L=6, 4x128 SiLU."""
        res = tuple(max(2, -(-int(n) // int(factor))) for n in dims)
        return cls(measure_kind=measure_kind, grid_resolution=res, precision=precision, **kw)


class NdfModel:
    """Instantiated NDF (model.py:105-142): host parameters + cached device state."""

    def __init__(self, spec: ModelSpec, grid_mu: np.ndarray, grid_nu: np.ndarray,
                 weights: list, biases: list, enc_mu=None, enc_nu=None, _shared=None):
        C = spec.features_per_level
        if spec.shared and grid_mu is not grid_nu:
            raise ConfigError("shared spec requires aliased grids")
        gshape = self.grid_shape(spec)
        for g in (grid_mu, grid_nu):
            if g.shape != gshape:
                raise ShapeError(f"latent grid shape {g.shape}, expected {gshape}")
        # encoders: (weights, biases) per branch; identity when encoder_layers == 0
        enc_mu = enc_mu if enc_mu is not None else ([], [])
        enc_nu = enc_nu if enc_nu is not None else enc_mu
        if spec.shared and enc_mu is not enc_nu:
            raise ConfigError("shared spec requires aliased encoders")
        ew = spec.encoder_widths()
        for ews, ebs in (enc_mu, enc_nu):
            if len(ews) != spec.encoder_layers or len(ebs) != len(ews):
                raise ConfigError("encoder layer count does not match spec")
            for i, (w, b) in enumerate(zip(ews, ebs)):
                if w.shape != (ew[i], ew[i + 1]) or b.shape != (ew[i + 1],):
                    raise ShapeError(f"encoder layer {i}: weight {w.shape} / bias {b.shape}")
        self.enc_mu = enc_mu
        self.enc_nu = enc_nu
        del C
        widths = spec.decoder_widths()
        if len(weights) != len(widths) - 1 or len(biases) != len(weights):
            raise ConfigError("decoder layer count does not match spec")
        for i, (w, b) in enumerate(zip(weights, biases)):
            if w.shape != (widths[i], widths[i + 1]) or b.shape != (widths[i + 1],):
                raise ShapeError(f"layer {i}: weight {w.shape} / bias {b.shape}")
        self.spec = spec
        self.grid_mu = grid_mu
        self.grid_nu = grid_nu
        self.weights = weights
        self.biases = biases
        self._dev = {}
        # parameter-version record shared by every NdfModel over the same host arrays
        # (with_precision copies): invalidate() on any of them retires all device copies
        self._shared = _shared if _shared is not None else {"version": 0}

    @staticmethod
    def grid_shape(spec: ModelSpec) -> tuple:
        """Latent array shape: (levels, 2^T, F) HashGrid tables for the reference family
        (encoding.py:127-133), (rz, ry, rx, C) for the dense level."""
        if spec.hash_grid:
            return (spec.levels, 1 << spec.log2_table_size, spec.features_per_level)
        rx, ry, rz = spec.latent_resolution
        return (rz, ry, rx, spec.features_per_level)

    @classmethod
    def build(cls, spec: ModelSpec, seed: int = 0, dtype=np.float32) -> "NdfModel":
        """Seeded init in the reference's RNG order (model.py:131-142; nn.py:76-93):
        grid_mu, enc_mu, [grid_nu, enc_nu], decoder; Kaiming-uniform weights, zero biases."""
        rng = np.random.default_rng(seed)
        s = spec.grid_init
        gshape = cls.grid_shape(spec)

        def mlp(widths):
            ws, bs = [], []
            for fan_in, fan_out in zip(widths[:-1], widths[1:]):
                bound = np.sqrt(6.0 / fan_in)
                ws.append(rng.uniform(-bound, bound, (fan_in, fan_out)).astype(dtype))
                bs.append(np.zeros(fan_out, dtype=dtype))
            return ws, bs

        grid_mu = rng.uniform(-s, s, size=gshape).astype(dtype)
        enc_mu = mlp(spec.encoder_widths())
        if spec.shared:
            grid_nu, enc_nu = grid_mu, enc_mu
        else:
            grid_nu = rng.uniform(-s, s, size=gshape).astype(dtype)
            enc_nu = mlp(spec.encoder_widths())
        ws, bs = mlp(spec.decoder_widths())
        return cls(spec, grid_mu, grid_nu, ws, bs, enc_mu, enc_nu)

    # -- parameters ---------------------------------------------------------

    def parameters(self) -> list:
        """Trainable arrays in canonical (NDFM) order (model.py:148-157)."""
        params = [self.grid_mu]
        if not self.spec.shared:
            params.append(self.grid_nu)
        for enc in ((self.enc_mu,) if self.spec.shared else (self.enc_mu, self.enc_nu)):
            for w, b in zip(*enc):
                params.extend((w, b))
        for w, b in zip(self.weights, self.biases):
            params.extend((w, b))
        return params

    def parameter_bytes(self) -> int:
        return int(sum(4 * p.size for p in self.parameters()))

    def validate_finite(self) -> None:
        for p in self.parameters():
            if not np.isfinite(p).all():
                raise ModelCorruptError("model contains non-finite parameters")

    def invalidate(self) -> None:
        """Make the parameters writable again and retire every device copy made from
        them (this model's and its with_precision siblings'): the next query re-validates
        (validate_finite, as the reference does per call, service.py:58-59) and re-uploads.

        Uploading freezes the host arrays (``writeable = False``): an in-place update --
        the reference's Adam.step writes model.parameters() in place (nn.py:197-214) --
        then raises instead of leaving the GPU copy silently stale."""
        self._shared["version"] += 1
        self._dev.clear()
        for p in self.parameters():
            try:
                p.flags.writeable = True
            except ValueError:
                pass               # a read-only base (e.g. a memory map) stays read-only

    def _freeze(self) -> None:
        for p in self.parameters():
            p.flags.writeable = False

    def swapped_roles(self) -> "NdfModel":
        """model.py:245-265 -- the (nu, mu) model sharing this model's parameters:
        ``swapped.forward(p1, p2) == self.forward(p2, p1)`` (exact for the commutative
        merges; concat reorders the first decoder layer's input blocks)."""
        spec = replace(self.spec, var_mu=self.spec.var_nu, var_nu=self.spec.var_mu)
        weights = list(self.weights)
        if self.spec.merge == "concat" and not self.spec.shared:
            half = self.spec.encoder_output_dim
            w0 = weights[0]
            weights[0] = np.concatenate([w0[half:], w0[:half]], axis=0)
        if self.spec.shared:
            return NdfModel(spec, self.grid_mu, self.grid_nu, weights, list(self.biases),
                            self.enc_mu, self.enc_nu)
        return NdfModel(spec, self.grid_nu, self.grid_mu, weights, list(self.biases),
                        self.enc_nu, self.enc_mu)

    def copy(self) -> "NdfModel":
        """model.py:267-277 -- independent parameter arrays (device copies are rebuilt)."""
        def cp(enc):
            return ([w.copy() for w in enc[0]], [b.copy() for b in enc[1]])
        grid_mu = self.grid_mu.copy()
        enc_mu = cp(self.enc_mu)
        if self.spec.shared:
            grid_nu, enc_nu = grid_mu, enc_mu
        else:
            grid_nu, enc_nu = self.grid_nu.copy(), cp(self.enc_nu)
        return NdfModel(self.spec, grid_mu, grid_nu, [w.copy() for w in self.weights],
                        [b.copy() for b in self.biases], enc_mu, enc_nu)

    def with_precision(self, precision: str) -> "NdfModel":
        """Same parameters, other query precision (shares host arrays)."""
        return NdfModel(replace(self.spec, precision=precision), self.grid_mu, self.grid_nu,
                        self.weights, self.biases, self.enc_mu, self.enc_nu, _shared=self._shared)

    # -- device state -------------------------------------------------------

    def device_state(self, device=None) -> "DeviceModel":
        dev = N.require_cuda(device)
        key = str(dev)
        st = self._dev.get(key)
        if st is None or st.version != self._shared["version"]:
            self.spec.check_gpu_supported()
            # validated once per upload; the arrays are frozen until invalidate(), so a
            # per-call re-check (service.py:58-59) could not find anything new
            self.validate_finite()
            st = DeviceModel(self, dev)
            self._freeze()
            st.version = self._shared["version"]
            self._dev[key] = st
        return st

    # -- embedding ----------------------------------------------------------

    def _branch(self, grid) -> int:
        if grid is self.grid_mu or (isinstance(grid, str) and grid == "mu"):
            return 0
        if grid is self.grid_nu or (isinstance(grid, str) and grid == "nu"):
            return 1
        tables = getattr(grid, "tables", None)          # a reference HashGrid
        if tables is not None:
            for b, mine in ((0, self.grid_mu), (1, self.grid_nu)):
                if tables is mine or (tables.shape == mine.shape and np.array_equal(tables, mine)):
                    return b
        raise ParameterError("grid must be this model's grid_mu / grid_nu (or 'mu' / 'nu')")

    def embed(self, grid, positions) -> np.ndarray:
        """model.py:169-177 -- [raw(3) | fourier(6L) | latent] per position, computed in
        fp64 and cast to fp32 on the GPU (ndf_embed_points), bit-identical to the reference.
        ``grid`` is this model's grid_mu / grid_nu (or "mu" / "nu")."""
        import torch
        branch = self._branch(grid)
        pos = np.atleast_2d(np.asarray(positions, dtype=np.float64))
        if pos.ndim != 2 or pos.shape[1] != 3:
            raise ShapeError(f"positions must be (B, 3), got {pos.shape}")
        st = self.device_state()
        out = torch.empty((pos.shape[0], self.spec.embed_dim), dtype=torch.float32,
                          device=st.device)
        if pos.shape[0]:
            dpos = torch.from_numpy(np.ascontiguousarray(pos)).to(st.device)
            N.call("ndf_embed_points", ctypes_ref(st.desc), branch, N.ptr(dpos), pos.shape[0],
                   N.ptr(out), N.stream_handle(st.device))
        return out.cpu().numpy()

    def embed_nodes(self, grid, dims, v0: int = 0, v1: int | None = None):
        """Embeddings of output-grid nodes [v0, v1) of ``dims`` (x fastest,
        measures.py:240-252) as a (v1 - v0, E) float32 CUDA tensor (ndf_embed_nodes)."""
        import torch
        branch = self._branch(grid)
        dims = tuple(int(d) for d in dims)
        if len(dims) != 3 or min(dims) < 1:
            raise ParameterError(f"grid dims must be >= 1, got {dims}")
        V = dims[0] * dims[1] * dims[2]
        v1 = V if v1 is None else int(v1)
        if not 0 <= v0 <= v1 <= V:
            raise ParameterError("vertex range out of bounds")
        st = self.device_state()
        out = torch.empty((v1 - v0, self.spec.embed_dim), dtype=torch.float32, device=st.device)
        N.call("ndf_embed_nodes", ctypes_ref(st.desc), branch, dims[0], dims[1], dims[2], v0, v1,
               N.ptr(out), N.stream_handle(st.device))
        return out

    # -- the reference's own model objects -------------------------------------

    @classmethod
    def from_reference(cls, ref, precision: str = "fp32") -> "NdfModel":
        """Convert the reference's ``ndf.model.NdfModel`` (HashGrid / Mlp objects,
        model.py:105-142) -- duck-typed on ``spec``, ``grid_mu.tables``, ``enc_mu.weights``
        and ``decoder.weights`` -- into this package's model.  The parameters are copied
        (a snapshot: training the reference object later does not touch this one; see
        ``as_model`` for the cached, change-detecting form).  A single dense level with
        no encoder becomes the dense layout, like an NDFM file (load_model); the
        reference family keeps its HashGrid tables and encoders (exact fp32 kernel)."""
        if isinstance(ref, NdfModel):
            return ref
        try:
            rspec = ref.spec
            names = [f for f in ModelSpec.__dataclass_fields__ if hasattr(rspec, f)]
            fields = {f: getattr(rspec, f) for f in names}
            acts = {ref.decoder.act}
            if ref.enc_mu.weights:
                acts |= {ref.enc_mu.act, ref.enc_nu.act}
        except AttributeError as exc:
            raise ConfigError(f"not a reference NdfModel: {exc}") from None
        if len(acts) != 1:
            raise ConfigError(f"mixed encoder / decoder activations {sorted(acts)} are not supported")
        fields.update(activation=acts.pop(), head="linear", precision=precision,
                      grid_resolution=None)
        spec = ModelSpec(**fields)
        cp = lambda a: np.array(a, dtype=np.float32, copy=True)   # noqa: E731
        t_mu = cp(ref.grid_mu.tables)
        t_nu = t_mu if spec.shared else cp(ref.grid_nu.tables)
        if not spec.hash_grid:
            rx, ry, rz = spec.latent_resolution
            C = spec.features_per_level
            t_mu = t_mu[0][: rx * ry * rz].reshape(rz, ry, rx, C).copy()
            t_nu = t_mu if spec.shared else t_nu[0][: rx * ry * rz].reshape(rz, ry, rx, C).copy()

        def mlp(m):
            return [cp(w) for w in m.weights], [cp(b) for b in m.biases]
        enc_mu = mlp(ref.enc_mu)
        enc_nu = enc_mu if spec.shared else mlp(ref.enc_nu)
        ws, bs = mlp(ref.decoder)
        return cls(spec, t_mu, t_nu, ws, bs, enc_mu, enc_nu)

    # -- forward ------------------------------------------------------------

    def forward(self, p_mu, p_nu, exact: bool = True) -> np.ndarray:
        """Batched dependence estimates (model.py:179-189), shape (B,) float32.

        Per-row results do not depend on the batch partitioning in either
        precision; ``exact`` is accepted for signature compatibility.
        """
        import torch
        p_mu = np.atleast_2d(np.asarray(p_mu, dtype=np.float64))
        p_nu = np.atleast_2d(np.asarray(p_nu, dtype=np.float64))
        for p in (p_mu, p_nu):
            if p.ndim != 2 or p.shape[1] != 3:
                raise ShapeError(f"positions must be (B, 3), got {p.shape}")
        if p_mu.shape[0] == p_nu.shape[0]:
            n_mu = n = p_mu.shape[0]
        elif p_mu.shape[0] == 1:
            n_mu, n = 1, p_nu.shape[0]
        elif p_nu.shape[0] == 1:           # broadcast nu: mirror of the mu broadcast
            p_nu = np.broadcast_to(p_nu, p_mu.shape)
            n_mu = n = p_mu.shape[0]
        else:
            raise ShapeError(f"cannot broadcast {p_mu.shape} against {p_nu.shape}")
        st = self.device_state()
        out = torch.empty(n, dtype=torch.float32, device=st.device)
        if n:
            pm = torch.from_numpy(np.ascontiguousarray(p_mu)).to(st.device)
            pn = torch.from_numpy(np.ascontiguousarray(p_nu)).to(st.device)
            N.call("ndf_query_points", ctypes_ref(st.desc), N.ptr(pm), n_mu, N.ptr(pn), n,
                   N.PREC[self.spec.precision], N.ptr(out), N.stream_handle(st.device))
        return out.cpu().numpy()

    def forward_pair(self, p_mu, p_nu) -> float:
        return float(self.forward(np.reshape(p_mu, (1, 3)), np.reshape(p_nu, (1, 3)))[0])


_FOREIGN = {}          # id(reference model) -> (fingerprint, converted NdfModel)


def _fingerprint(arrays) -> tuple:
    """Cheap content key of a parameter list: identity, shape and two 64-bit folds of
    the bytes (sum and xor) -- an in-place training step changes it."""
    key = []
    for a in arrays:
        a = np.ascontiguousarray(a)
        u = a.reshape(-1).view(np.uint8)
        pad = (-u.size) % 8
        if pad:
            u = np.concatenate([u, np.zeros(pad, np.uint8)])
        w = u.view(np.uint64)
        key.append((a.shape, str(a.dtype), int(np.add.reduce(w, dtype=np.uint64)),
                    int(np.bitwise_xor.reduce(w)) if w.size else 0))
    return tuple(key)


def as_model(model, precision: str | None = None) -> NdfModel:
    """This package's NdfModel for ``model``: itself, or the conversion of a reference
    ``ndf.model.NdfModel`` (NdfModel.from_reference), cached per object and rebuilt
    when the reference's parameters change (the reference trains in place,
    nn.py:197-214).  ``precision`` applies to converted models (default fp32, the
    reference's own arithmetic)."""
    if isinstance(model, NdfModel):
        return model
    import weakref
    params = model.parameters() if hasattr(model, "parameters") else None
    if params is None:
        raise ConfigError(f"not an NDF model: {type(model).__name__}")
    fp = _fingerprint(params)
    key = (id(model), precision or "fp32")
    hit = _FOREIGN.get(key)
    if hit is not None and hit[0] == fp and hit[2]() is model:
        return hit[1]
    conv = NdfModel.from_reference(model, precision or "fp32")
    try:
        ref = weakref.ref(model)
        weakref.finalize(model, _FOREIGN.pop, key, None)
    except TypeError:                      # not weak-referenceable: do not cache
        return conv
    _FOREIGN[key] = (fp, conv, ref)
    return conv


def ctypes_ref(desc):
    import ctypes
    return ctypes.byref(desc)


class DeviceModel:
    """HBM-resident copy of an NdfModel: latent grids, fp32 params, packed bf16 blob."""

    def __init__(self, model: NdfModel, device):
        import torch
        spec = model.spec
        self.device = device
        self.grid_mu = torch.from_numpy(np.array(model.grid_mu, dtype=np.float32, copy=True)).to(device)
        self.grid_nu = self.grid_mu if spec.shared else torch.from_numpy(
            np.array(model.grid_nu, dtype=np.float32, copy=True)).to(device)
        def flat(ws, bs):
            return np.concatenate([np.concatenate([w.ravel(), b.ravel()])
                                   for w, b in zip(ws, bs)]).astype(np.float32)

        self.params = torch.from_numpy(flat(model.weights, model.biases)).to(device)
        widths = spec.decoder_widths()
        d = N.ModelDesc()
        d.fourier_octaves = spec.fourier_octaves
        d.grid_channels = spec.features_per_level
        for i, r in enumerate(spec.latent_resolution):
            d.grid_res[i] = r
        self.enc_mu = self.enc_nu = None
        if spec.hash_grid:
            d.grid_levels = spec.levels
            d.grid_log2_table = spec.log2_table_size
            for i, r in enumerate(spec.level_resolutions()):
                d.grid_level_res[i] = r
            d.enc_layers = spec.encoder_layers
            for i, w in enumerate(spec.encoder_widths()):
                d.enc_widths[i] = w
            if spec.encoder_layers:
                self.enc_mu = torch.from_numpy(flat(*model.enc_mu)).to(device)
                self.enc_nu = self.enc_mu if spec.shared else torch.from_numpy(
                    flat(*model.enc_nu)).to(device)
                d.enc_mu = self.enc_mu.data_ptr()
                d.enc_nu = self.enc_nu.data_ptr()
        d.merge = N.MERGE[spec.merge]
        d.activation = N.ACT[spec.activation]
        d.head = N.HEAD[spec.head_kind]
        d.n_layers = len(widths) - 1
        for i, w in enumerate(widths):
            d.widths[i] = w
        d.grid_mu = self.grid_mu.data_ptr()
        d.grid_nu = self.grid_nu.data_ptr()
        d.params_f32 = self.params.data_ptr()
        d.params_tc = None
        d.tc_format = N.PREC["fp16"] if spec.precision == "fp16" else N.PREC["bf16"]
        self.blob = None
        lib = N.load_library()
        nbytes = int(lib.ndf_tc_blob_bytes(ctypes_ref(d)))
        if nbytes:
            self.blob = torch.empty(nbytes, dtype=torch.uint8, device=device)
            N.call("ndf_tc_pack", ctypes_ref(d), N.ptr(self.blob), nbytes, N.stream_handle(device))
            d.params_tc = self.blob.data_ptr()
        elif spec.precision in ("bf16", "fp16"):
            raise ConfigError("model is outside the tcgen05 kernel envelope (L=6, C=16, "
                              "hidden width 128, input width <= 128); use precision='fp32'")
        self.desc = d
        self.desc_ref = ctypes_ref(d)      # reused by every query call


# ---------------------------------------------------------------------------
# NDFM container (model.py:315-387)


def save_model(model: NdfModel, path) -> None:
    spec = model.spec
    header = dict(asdict(spec))
    header["shared_encoder"] = spec.shared
    header["grid_resolution"] = None if spec.hash_grid else list(spec.latent_resolution)
    header["encoder_widths"] = spec.encoder_widths()
    header["decoder_widths"] = spec.decoder_widths()
    raw_header = json.dumps(header, sort_keys=True).encode("utf-8")
    with open(path, "wb") as fh:
        fh.write(NDFM_MAGIC)
        fh.write(struct.pack("<2I", NDFM_VERSION, len(raw_header)))
        fh.write(raw_header)
        for p in model.parameters():
            fh.write(np.ascontiguousarray(p, dtype="<f4").tobytes())


def load_model(path) -> NdfModel:
    """Read an NDFM container (ours, or an unmodified reference one, model.py:331-387).

    Reference files (no ``grid_resolution`` key) store the hash tables as
    (levels, 2^T, F), then the encoder(s), then the decoder, all SnakeAlt with a
    linear output (model.py:131-142, nn.py:136).  The reference family loads as
    is (HashGrid + encoders, exact fp32 path); a single dense level without
    encoder is converted to the dense layout: its first res^3 rows are the grid
    in ix + res*(iy + res*iz) order (encoding.py:97-98).
    """
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != NDFM_MAGIC:
            raise FormatError(f"bad magic {magic!r}, expected {NDFM_MAGIC!r}")
        head = fh.read(8)
        if len(head) != 8:
            raise FormatError("truncated NDFM header")
        version, header_len = struct.unpack("<2I", head)
        if version != NDFM_VERSION:
            raise FormatError(f"unsupported NDFM version {version}")
        raw_header = fh.read(header_len)
        if len(raw_header) != header_len:
            raise FormatError("truncated NDFM descriptor")
        try:
            header = json.loads(raw_header.decode("utf-8"))
        except (UnicodeDecodeError, json.JSONDecodeError) as exc:
            raise FormatError(f"bad NDFM descriptor: {exc}") from exc
        blob = fh.read()
    values = np.frombuffer(blob, dtype="<f4")
    reference_file = "grid_resolution" not in header
    fields = {k: header[k] for k in ModelSpec.__dataclass_fields__ if k in header}
    if reference_file:
        fields.update(activation="snake_alt", head="linear")
    if fields.get("grid_resolution") is not None:
        fields["grid_resolution"] = tuple(fields["grid_resolution"])
    spec = ModelSpec(**fields)
    cursor = 0

    def take(shape):
        nonlocal cursor
        n = int(np.prod(shape))
        if cursor + n > values.size:
            raise FormatError("NDFM payload truncated")
        out = values[cursor:cursor + n].reshape(shape).copy()
        cursor += n
        return out

    def take_mlp(widths):
        ws, bs = [], []
        for fan_in, fan_out in zip(widths[:-1], widths[1:]):
            ws.append(take((fan_in, fan_out)))
            bs.append(take((fan_out,)))
        return ws, bs

    rx, ry, rz = spec.latent_resolution
    C = spec.features_per_level
    if spec.hash_grid:
        gshape = NdfModel.grid_shape(spec)
        t_mu = take(gshape)
        t_nu = t_mu if spec.shared else take(gshape)
    elif reference_file:
        T = 1 << spec.log2_table_size
        t_mu = take((1, T, C))[0][: rx ** 3].reshape(rz, ry, rx, C).copy()
        t_nu = t_mu if spec.shared else take((1, T, C))[0][: rx ** 3].reshape(rz, ry, rx, C).copy()
    else:
        t_mu = take((rz, ry, rx, C))
        t_nu = t_mu if spec.shared else take((rz, ry, rx, C))
    enc_mu = take_mlp(spec.encoder_widths())
    enc_nu = enc_mu if spec.shared else take_mlp(spec.encoder_widths())
    ws, bs = take_mlp(spec.decoder_widths())
    if cursor != values.size:
        raise FormatError(f"NDFM payload has {values.size - cursor} stray values")
    model = NdfModel(spec, t_mu, t_nu, ws, bs, enc_mu, enc_nu)
    model.validate_finite()
    return model
