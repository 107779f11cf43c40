"""NDF model: spec, parameters, GPU-resident state, NDFM IO (drop-in for model.py).

``ModelSpec`` keeps every field of the reference (``model.py:29-102``) and
adds the BASELINE.json architecture knobs: a dense
anisotropic latent grid (``grid_resolution``), the ``sum_absdiff`` merge,
SiLU hidden activations, a tanh/softplus ``head`` and the query
``precision`` ("fp32" = exact SIMT kernel, "bf16" = tcgen05 kernel).

The GPU path covers the encoder-less family (``encoder_layers == 0``) with one
dense latent level per branch -- BASELINE's architecture and the reference's
``encoder_layers=0`` single-dense-level ablation.  Multi-level hashed grids
and encoder MLPs (the reference default) are SURVEY row F3 ("next") and are
rejected with ConfigError rather than silently evaluated on the CPU.
"""

from __future__ import annotations

import json
import struct
from dataclasses import asdict, dataclass, replace

import numpy as np

from . import _native as N
from .errors import ConfigError, FormatError, ModelCorruptError, ShapeError

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
        if self.encoder_layers != 0:
            raise ConfigError("encoder MLPs (encoder_layers > 0) are not on the GPU path yet "
                              "(SURVEY row F3)")
        if self.levels != 1:
            raise ConfigError("multi-level hash grids are not on the GPU path yet (SURVEY row F3)")
        if self.grid_resolution is None:
            r = self.latent_resolution[0]
            if r ** 3 > (1 << self.log2_table_size):
                raise ConfigError("hashed (res^3 > 2^T) levels are not on the GPU path yet")
        widths = self.decoder_widths()
        if len(widths) - 1 > N.NDF_MAX_LAYERS or max(widths) > N.NDF_MAX_WIDTH:
            raise ConfigError("decoder exceeds the kernel envelope (<= 8 layers, width <= 256)")
        if self.fourier_octaves > 12 or self.features_per_level > 64:
            raise ConfigError("encoder exceeds the kernel envelope (L <= 12, C <= 64)")

    @classmethod
    def baseline(cls, dims, factor: int, measure_kind: str = "pearson",
                 precision: str = "fp32", **kw) -> "ModelSpec":
        """BASELINE.json model: 16-ch latent at 1/factor resolution, L=6, 4x128 SiLU."""
        res = tuple(max(2, -(-int(n) // int(factor))) for n in dims)
        return cls(measure_kind=measure_kind, grid_resolution=res, precision=precision, **kw)


class NdfModel:
    """Instantiated NDF (model.py:105-142): host parameters + cached device state."""

    def __init__(self, spec: ModelSpec, grid_mu: np.ndarray, grid_nu: np.ndarray,
                 weights: list, biases: list):
        rx, ry, rz = spec.latent_resolution
        C = spec.features_per_level
        if spec.shared and grid_mu is not grid_nu:
            raise ConfigError("shared spec requires aliased grids")
        for g in (grid_mu, grid_nu):
            if g.shape != (rz, ry, rx, C):
                raise ShapeError(f"latent grid shape {g.shape}, expected {(rz, ry, rx, C)}")
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

    @classmethod
    def build(cls, spec: ModelSpec, seed: int = 0, dtype=np.float32) -> "NdfModel":
        """Seeded init in the reference's RNG order (model.py:131-142; nn.py:76-93)."""
        rng = np.random.default_rng(seed)
        rx, ry, rz = spec.latent_resolution
        C = spec.features_per_level
        s = spec.grid_init
        grid_mu = rng.uniform(-s, s, size=(rz, ry, rx, C)).astype(dtype)
        grid_nu = grid_mu if spec.shared else rng.uniform(-s, s, size=(rz, ry, rx, C)).astype(dtype)
        widths = spec.decoder_widths()
        ws, bs = [], []
        for fan_in, fan_out in zip(widths[:-1], widths[1:]):
            bound = np.sqrt(6.0 / fan_in)
            ws.append(rng.uniform(-bound, bound, (fan_in, fan_out)).astype(dtype))
            bs.append(np.zeros(fan_out, dtype=dtype))
        return cls(spec, grid_mu, grid_nu, ws, bs)

    # -- parameters ---------------------------------------------------------

    def parameters(self) -> list:
        """Trainable arrays in canonical (NDFM) order (model.py:148-157)."""
        params = [self.grid_mu]
        if not self.spec.shared:
            params.append(self.grid_nu)
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
        """Drop cached device copies (call after mutating parameters in place)."""
        self._dev.clear()

    def with_precision(self, precision: str) -> "NdfModel":
        """Same parameters, other query precision (shares host arrays)."""
        return NdfModel(replace(self.spec, precision=precision), self.grid_mu, self.grid_nu,
                        self.weights, self.biases)

    # -- device state -------------------------------------------------------

    def device_state(self, device=None) -> "DeviceModel":
        dev = N.require_cuda(device)
        key = str(dev)
        if key not in self._dev:
            self.spec.check_gpu_supported()
            self.validate_finite()        # once per upload (failure detection)
            self._dev[key] = DeviceModel(self, dev)
        return self._dev[key]

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


def ctypes_ref(desc):
    import ctypes
    return ctypes.byref(desc)


class DeviceModel:
    """HBM-resident copy of an NdfModel: latent grids, fp32 params, packed bf16 blob."""

    def __init__(self, model: NdfModel, device):
        import torch
        spec = model.spec
        self.device = device
        self.grid_mu = torch.from_numpy(np.ascontiguousarray(model.grid_mu, np.float32)).to(device)
        self.grid_nu = self.grid_mu if spec.shared else torch.from_numpy(
            np.ascontiguousarray(model.grid_nu, np.float32)).to(device)
        flat = np.concatenate([np.concatenate([w.ravel(), b.ravel()])
                               for w, b in zip(model.weights, model.biases)]).astype(np.float32)
        self.params = torch.from_numpy(flat).to(device)
        widths = spec.decoder_widths()
        d = N.ModelDesc()
        d.fourier_octaves = spec.fourier_octaves
        d.grid_channels = spec.features_per_level
        for i, r in enumerate(spec.latent_resolution):
            d.grid_res[i] = r
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


# ---------------------------------------------------------------------------
# NDFM container (model.py:315-387)


def save_model(model: NdfModel, path) -> None:
    spec = model.spec
    header = dict(asdict(spec))
    header["shared_encoder"] = spec.shared
    header["grid_resolution"] = list(spec.latent_resolution)
    header["encoder_widths"] = [spec.embed_dim]
    header["decoder_widths"] = spec.decoder_widths()
    raw_header = json.dumps(header, sort_keys=True).encode("utf-8")
    with open(path, "wb") as fh:
        fh.write(NDFM_MAGIC)
        fh.write(struct.pack("<2I", NDFM_VERSION, len(raw_header)))
        fh.write(raw_header)
        for p in model.parameters():
            fh.write(np.ascontiguousarray(p, dtype="<f4").tobytes())


def load_model(path) -> NdfModel:
    """Read an NDFM container (ours, or a reference one inside the GPU envelope).

    Reference files (no ``grid_resolution`` key) store the hash table as
    (levels, 2^T, F); with levels == 1 and a dense level (res^3 <= 2^T) the
    first res^3 rows are the dense grid in ix + res*(iy + res*iz) order
    (encoding.py:97-98), and the decoder uses SnakeAlt with a linear output
    (model.py:141, nn.py:136).
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
    if spec.encoder_layers != 0 or spec.levels != 1:
        raise ConfigError("NDFM model uses encoder MLPs / multi-level grids: not on the GPU path")
    cursor = 0

    def take(shape):
        nonlocal cursor
        n = int(np.prod(shape))
        if cursor + n > values.size:
            raise FormatError("NDFM payload truncated")
        out = values[cursor:cursor + n].reshape(shape).copy()
        cursor += n
        return out

    rx, ry, rz = spec.latent_resolution
    C = spec.features_per_level
    if reference_file:
        T = 1 << spec.log2_table_size
        if rx ** 3 > T:
            raise ConfigError("reference NDFM uses a hashed level: not on the GPU path")
        t_mu = take((1, T, C))[0][: rx ** 3].reshape(rz, ry, rx, C).copy()
        t_nu = t_mu if spec.shared else take((1, T, C))[0][: rx ** 3].reshape(rz, ry, rx, C).copy()
    else:
        t_mu = take((rz, ry, rx, C))
        t_nu = t_mu if spec.shared else take((rz, ry, rx, C))
    widths = spec.decoder_widths()
    ws, bs = [], []
    for fan_in, fan_out in zip(widths[:-1], widths[1:]):
        ws.append(take((fan_in, fan_out)))
        bs.append(take((fan_out,)))
    if cursor != values.size:
        raise FormatError(f"NDFM payload has {values.size - cursor} stray values")
    model = NdfModel(spec, t_mu, t_nu, ws, bs)
    model.validate_finite()
    return model
