"""ctypes binding of libndf_b200.so (the C-ABI declared in include/ndf_b200.h).

This is the only door to the compute path: if the shared library or a CUDA
device is missing, calls raise ``DeviceError`` -- there is no CPU fallback.
PyTorch is used purely as plumbing: device memory (tensors), the current
stream handle, and ``torch.distributed`` elsewhere.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ConfigError, DeviceError, ParameterError, ShapeError

HERE = os.path.dirname(os.path.abspath(__file__))
# NDF_LIB_PATH points timing experiments at a variant build (tools/build_variants.sh)
# without touching the product library next to this file.
LIB_PATH = os.environ.get("NDF_LIB_PATH") or os.path.join(HERE, "libndf_b200.so")

NDF_MAX_LAYERS = 8
NDF_MAX_WIDTH = 256
NDF_MAX_LEVELS = 16
NDF_ABI_VERSION = 3

MERGE = {"multiply": 0, "concat": 1, "add": 2, "absdiff": 3, "sum_absdiff": 4}
ACT = {"relu": 0, "snake": 1, "snake_alt": 2, "silu": 3}
HEAD = {"linear": 0, "tanh": 1, "softplus": 2}
PREC = {"fp32": 0, "bf16": 1, "fp16": 2}

_c_p = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f64 = ctypes.c_double


class ModelDesc(ctypes.Structure):
    """Mirror of ``ndf_model_desc``."""

    _fields_ = [
        ("fourier_octaves", _i32),
        ("grid_channels", _i32),
        ("grid_res", _i32 * 3),
        ("merge", _i32),
        ("activation", _i32),
        ("head", _i32),
        ("n_layers", _i32),
        ("widths", _i32 * (NDF_MAX_LAYERS + 1)),
        ("tc_format", _i32),
        ("grid_mu", _c_p),
        ("grid_nu", _c_p),
        ("params_f32", _c_p),
        ("params_tc", _c_p),
        # ABI 2: reference HashGrid + encoder MLPs
        ("grid_levels", _i32),
        ("grid_log2_table", _i32),
        ("grid_level_res", _i32 * NDF_MAX_LEVELS),
        ("enc_layers", _i32),
        ("enc_widths", _i32 * (NDF_MAX_LAYERS + 1)),
        ("enc_mu", _c_p),
        ("enc_nu", _c_p),
    ]


# name -> (restype, argtypes)
SIGNATURES = {
    "ndf_abi_version": (_i32, []),
    "ndf_last_error": (ctypes.c_char_p, []),
    "ndf_device_sm_count": (_i32, []),
    "ndf_tc_blob_bytes": (ctypes.c_size_t, [ctypes.POINTER(ModelDesc)]),
    "ndf_tc_pack": (ctypes.c_int, [ctypes.POINTER(ModelDesc), _c_p, ctypes.c_size_t, _c_p]),
    "ndf_query_grid": (ctypes.c_int, [ctypes.POINTER(ModelDesc), _f64, _f64, _f64, _i32, _i32,
                                      _i32, _i32, _i64, _i64, _i32, _c_p, _c_p]),
    "ndf_query_grid_stats": (ctypes.c_int, [ctypes.POINTER(ModelDesc), _f64, _f64, _f64, _i32,
                                            _i32, _i32, _i32, _i64, _i64, _i32, _c_p, _c_p,
                                            _c_p]),
    "ndf_query_points": (ctypes.c_int, [ctypes.POINTER(ModelDesc), _c_p, _i64, _c_p, _i64, _i32,
                                        _c_p, _c_p]),
    "ndf_embed_nodes": (ctypes.c_int, [ctypes.POINTER(ModelDesc), _i32, _i32, _i32, _i32, _i64,
                                       _i64, _c_p, _c_p]),
    "ndf_embed_points": (ctypes.c_int, [ctypes.POINTER(ModelDesc), _i32, _c_p, _i64, _c_p, _c_p]),
    "ndf_query_grid_multi": (ctypes.c_int, [ctypes.POINTER(ModelDesc), _c_p, _i32, _i32, _i32,
                                            _i32, _i32, _i64, _i64, _c_p, _i64, _c_p]),
    "ndf_sample_many": (ctypes.c_int, [_c_p, _i32, _i32, _i32, _i32, _c_p, _i64, _c_p, _c_p]),
    "ndf_sample_many_vm": (ctypes.c_int, [_c_p, _i32, _i32, _i32, _i32, _c_p, _i64, _c_p, _c_p]),
    "ndf_sample_many_ld": (ctypes.c_int, [_c_p, _i32, _i64, _i64, _i32, _i32, _i32, _c_p, _i64,
                                          _c_p, _c_p]),
    "ndf_pearson_field": (ctypes.c_int, [_c_p, _i32, _i64, _i64, _c_p, _i64, _i64, _c_p, _c_p]),
    "ndf_field_export": (ctypes.c_int, [_c_p, _c_p, _i64, _c_p, _c_p, _i32, _c_p]),
    "ndf_zscore": (ctypes.c_int, [_c_p, _i32, _i64, _i64, _i64, _c_p, _c_p, _c_p]),
    "ndf_pearson_gemv": (ctypes.c_int, [_c_p, _c_p, _i32, _i64, _c_p, _i32, _i64, _i64, _c_p,
                                        _c_p]),
    "ndf_pearson_rows": (ctypes.c_int, [_c_p, _i64, _c_p, _i32, _i64, _c_p, _c_p]),
    "ndf_vertex_major": (ctypes.c_int, [_c_p, _i32, _i64, _c_p, _c_p]),
    "ndf_pearson_pairs": (ctypes.c_int, [_c_p, _i32, _i64, _c_p, _c_p, _i64, _c_p, _c_p]),
    "ndf_ksg_ref_nodes": (ctypes.c_int, [_c_p, _i32, _i64, _c_p, _i64, _i64, _i32, _c_p, _c_p,
                                         _f64, _c_p, _c_p, _c_p, _c_p, _c_p]),
    "ndf_ksg_rows": (ctypes.c_int, [_c_p, _i64, _c_p, _i32, _i64, _i32, _c_p, _c_p, _f64, _c_p,
                                    _c_p, _c_p, _c_p, _c_p]),
    "ndf_ksg_pairs": (ctypes.c_int, [_c_p, _i32, _i64, _c_p, _c_p, _i64, _i32, _c_p, _c_p, _f64,
                                     _c_p, _c_p, _c_p, _c_p, _c_p]),
    "ndf_launch_count": (_i64, [_i32]),
}

_lock = threading.Lock()
_lib = None


def load_library(path: str = LIB_PATH):
    """Load (once) and type the shared library; raises DeviceError if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceError(
                f"{path} is not built; run `python -m paper_2307_02203_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.ndf_abi_version() != NDF_ABI_VERSION:
            raise DeviceError("libndf_b200 ABI version mismatch")
        _lib = lib
        return lib


def check(status: int) -> None:
    """Map an ndf_status to the reference's exception classes."""
    if status == 0:
        return
    msg = _lib.ndf_last_error().decode("utf-8", "replace") if _lib else "unknown error"
    if status in (1, 6):
        raise ParameterError(msg)
    if status == 2:
        raise ShapeError(msg)
    if status in (3, 5):
        raise ConfigError(msg)
    raise DeviceError(msg)


_CHECKED_DEVICES = {}


def require_cuda(device=None):
    """Return a torch CUDA device or raise DeviceError (no CPU fallback).  A device
    that passed the checks once is cached (this sits on every query's host path)."""
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device available: the NDF B200 kernels need an sm_100a GPU")
    key = torch.cuda.current_device() if device is None else device
    dev = _CHECKED_DEVICES.get(key) if isinstance(key, (int, str)) else None
    if dev is not None:
        return dev
    dev = torch.device(device) if device is not None else torch.device("cuda", key)
    if dev.type != "cuda":
        raise DeviceError(f"device {dev} is not a CUDA device")
    major, _ = torch.cuda.get_device_capability(dev)
    if major < 10:
        raise DeviceError("libndf_b200 is compiled for sm_100a (B200) only")
    if isinstance(key, (int, str)):
        _CHECKED_DEVICES[key] = dev
    return dev


def stream_handle(device=None):
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def ptr(t) -> ctypes.c_void_p:
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return ctypes.c_void_p(0)
    return ctypes.c_void_p(t.data_ptr())


def call(name: str, *args) -> None:
    lib = load_library()
    check(getattr(lib, name)(*args))


def launch_count(reset: bool = False) -> int:
    return int(load_library().ndf_launch_count(1 if reset else 0))
