"""ctypes binding of libssimk.so (include/ssimk.h) plus device marshalling.

This is the only module that touches the native library.  There is no CPU
fallback: if the library is missing or no CUDA device is present, every
scoring entry point raises ``EngineUnavailable`` (the engine must fail loudly
rather than silently compute on the host).
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path
from typing import Optional

import numpy as np

from .errors import (
    EngineUnavailable,
    SsimkitError,
    TooManyLevels,
    TooSmall,
    ValidationError,
    WindowLargerThanImage,
)

# SSK_LIBRARY overrides the library path (tools/sync_stress.py loads the stress build this way)
LIB_PATH = Path(os.environ.get("SSK_LIBRARY") or Path(__file__).resolve().parent / "_lib" / "libssimk.so")

# enums (include/ssimk.h)
U8, U16, U32, F32, F64 = 1, 2, 3, 4, 5
RECT, GAUSS = 1, 2
WANT_Q, WANT_L, WANT_CS, MAP_TERMS, MAP_STATS, WANT_Q2, MAP_F64 = 1, 2, 4, 8, 16, 32, 64
PW_V, PW_SQDEV, PW_ABSDEV_P, PW_ONEMINUS_P, PW_DW_NUM, PW_PP, PW_LW = range(7)
E_ARG, E_WINDOW, E_SHAPE, E_WORKSPACE, E_ALIGN, E_CUDA, E_LEVELS, E_TOO_SMALL = range(-1, -9, -1)

ABI_VERSION = 9
GAUSS_MAX_K = 255  # SSK_GAUSS_MAX_K

EXPORTED_SYMBOLS = (
    "ssk_abi_version",
    "ssk_stats_from_sums",
    "ssk_pairwise_workspace_bytes",
    "ssk_pairwise_sum",
    "ssk_term_maps",
    "ssk_divide",
    "ssk_strerror",
    "ssk_ssim_workspace_bytes",
    "ssk_msssim_workspace_bytes",
    "ssk_ssim",
    "ssk_box_window_sums",
    "ssk_integral_tables",
    "ssk_downsample",
    "ssk_msssim",
    "ssk_volume_update",
    "ssk_volume_refresh",
    "ssk_volume_workspace_bytes",
    "ssk_volume_ssim",
    "ssk_box_downsample",
    "ssk_pool_workspace_bytes",
    "ssk_pool_spatial",
    "ssk_pool_moments",
    "ssk_color_convert",
    "ssk_qssim_workspace_bytes",
    "ssk_qssim",
    "ssk_delta_e_workspace_bytes",
    "ssk_delta_e",
    "ssk_host_register",
    "ssk_host_unregister",
    "ssk_launch_count",
    "ssk_probe_fp32_tflops",
)

SPACE_RGB, SPACE_YCBCR = 1, 2
CONV_RGB, CONV_YCBCR, CONV_LUMA, CONV_HUE, CONV_LAB_EMBED = 1, 2, 3, 4, 5

# spatial pooler kinds (SSK_POOL_*), in SPATIAL_KINDS order of src/pooling.py:29
POOL_KINDS = {"am": 0, "cov": 1, "md": 2, "fns": 3, "dw": 4, "mink": 5, "lw": 6, "pp": 7}
POOL_PCTL = 8  # np.percentile(v, ps) itself (SSK_POOL_PCTL)


class Planes(ctypes.Structure):
    _fields_ = [
        ("ref", ctypes.c_void_p),
        ("dist", ctypes.c_void_p),
        ("dtype", ctypes.c_int32),
        ("scale_log2", ctypes.c_int32),
        ("n", ctypes.c_int32),
        ("h", ctypes.c_int32),
        ("w", ctypes.c_int32),
        ("bit_depth", ctypes.c_int32),
        ("row_pitch", ctypes.c_int64),
        ("frame_pitch", ctypes.c_int64),
    ]


class Volume(ctypes.Structure):
    _fields_ = [
        ("planes", ctypes.c_void_p),
        ("is_float", ctypes.c_int32),
        ("h", ctypes.c_int32),
        ("w", ctypes.c_int32),
        ("depth", ctypes.c_int32),
        ("pitch", ctypes.c_int64),
    ]


class Maps(ctypes.Structure):
    _fields_ = [
        ("values", ctypes.c_void_p),
        ("aux", ctypes.c_void_p),
        ("dtype", ctypes.c_int32),
        ("n", ctypes.c_int32),
        ("h", ctypes.c_int32),
        ("w", ctypes.c_int32),
        ("row_pitch", ctypes.c_int64),
        ("frame_pitch", ctypes.c_int64),
        ("aux_row_pitch", ctypes.c_int64),
        ("aux_frame_pitch", ctypes.c_int64),
    ]


class Pooler(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
        ("p", ctypes.c_double),
        ("o", ctypes.c_double),
        ("a", ctypes.c_double),
        ("b", ctypes.c_double),
        ("ps", ctypes.c_double),
        ("rs", ctypes.c_double),
    ]


class Color(ctypes.Structure):
    _fields_ = [
        ("ch", ctypes.c_void_p * 3),
        ("dtype", ctypes.c_int32),
        ("space", ctypes.c_int32),
        ("subsampling", ctypes.c_int32),
        ("n", ctypes.c_int32),
        ("h", ctypes.c_int32),
        ("w", ctypes.c_int32),
        ("bit_depth", ctypes.c_int32),
        ("row_pitch", ctypes.c_int64 * 3),
        ("frame_pitch", ctypes.c_int64 * 3),
    ]


class Window(ctypes.Structure):
    _fields_ = [
        ("shape", ctypes.c_int32),
        ("k", ctypes.c_int32),
        ("stride", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
        ("c1", ctypes.c_double),
        ("c2", ctypes.c_double),
        ("sigma", ctypes.c_double),
        ("taps", ctypes.c_float * 32),
    ]


_lib: Optional[ctypes.CDLL] = None
_lib_lock = threading.Lock()


def load_library(path: Path = LIB_PATH) -> ctypes.CDLL:
    """Load and type the C ABI (works without a GPU: no CUDA call is made)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not path.exists():
            raise EngineUnavailable(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(str(path))
        vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
        pP, pW = ctypes.POINTER(Planes), ctypes.POINTER(Window)
        lib.ssk_abi_version.restype = i32
        lib.ssk_strerror.restype = ctypes.c_char_p
        lib.ssk_strerror.argtypes = [i32]
        lib.ssk_ssim_workspace_bytes.restype = sz
        lib.ssk_ssim_workspace_bytes.argtypes = [pP, pW]
        lib.ssk_msssim_workspace_bytes.restype = sz
        lib.ssk_msssim_workspace_bytes.argtypes = [pP, pW, i32]
        lib.ssk_pairwise_workspace_bytes.restype = sz
        lib.ssk_pairwise_workspace_bytes.argtypes = [ctypes.POINTER(Maps)]
        lib.ssk_pairwise_sum.restype = i32
        lib.ssk_pairwise_sum.argtypes = [ctypes.POINTER(Maps), i32, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_double, vp, vp, vp, sz, vp]
        lib.ssk_stats_from_sums.restype = i32
        lib.ssk_stats_from_sums.argtypes = [vp, vp, vp, vp, vp, i64, ctypes.c_double, vp, vp]
        lib.ssk_term_maps.restype = i32
        lib.ssk_term_maps.argtypes = [vp, vp, vp, vp, vp, i64, ctypes.c_double, ctypes.c_double, vp, vp]
        lib.ssk_divide.restype = i32
        lib.ssk_divide.argtypes = [vp, i64, ctypes.c_double, vp, vp]
        lib.ssk_ssim.restype = i32
        lib.ssk_ssim.argtypes = [pP, pW, i32, vp, vp, vp, sz, vp]
        lib.ssk_box_window_sums.restype = i32
        lib.ssk_box_window_sums.argtypes = [pP, i32, i32, vp, vp, sz, vp]
        lib.ssk_integral_tables.restype = i32
        lib.ssk_integral_tables.argtypes = [pP, vp, vp]
        lib.ssk_downsample.restype = i32
        lib.ssk_downsample.argtypes = [pP, vp, vp, i32, i64, i64, vp]
        lib.ssk_msssim.restype = i32
        lib.ssk_msssim.argtypes = [pP, pW, i32, ctypes.POINTER(ctypes.c_double), i32, vp, vp, vp, vp, sz, vp]
        pV = ctypes.POINTER(Volume)
        lib.ssk_volume_update.restype = i32
        lib.ssk_volume_update.argtypes = [pV, vp, vp, vp, vp, i32, i64, i32, vp]
        lib.ssk_volume_refresh.restype = i32
        lib.ssk_volume_refresh.argtypes = [pV, ctypes.POINTER(vp), ctypes.POINTER(vp), i32, i32, i64, vp]
        lib.ssk_volume_workspace_bytes.restype = sz
        lib.ssk_volume_workspace_bytes.argtypes = [pV, pW]
        lib.ssk_volume_ssim.restype = i32
        lib.ssk_volume_ssim.argtypes = [pV, pW, i32, vp, vp, vp, sz, vp]
        lib.ssk_box_downsample.restype = i32
        lib.ssk_box_downsample.argtypes = [pP, i32, vp, vp, i32, i64, i64, vp]
        pM, pQ = ctypes.POINTER(Maps), ctypes.POINTER(Pooler)
        lib.ssk_pool_workspace_bytes.restype = sz
        lib.ssk_pool_workspace_bytes.argtypes = [pM, pQ]
        lib.ssk_pool_spatial.restype = i32
        lib.ssk_pool_spatial.argtypes = [pM, pQ, vp, vp, vp, sz, vp]
        lib.ssk_pool_moments.restype = i32
        lib.ssk_pool_moments.argtypes = [vp, i32, ctypes.c_double, pQ, vp, vp, vp]
        pC, pD = ctypes.POINTER(Color), ctypes.POINTER(ctypes.c_double)
        lib.ssk_color_convert.restype = i32
        lib.ssk_color_convert.argtypes = [pC, i32, vp, i64, i64, vp]
        lib.ssk_qssim_workspace_bytes.restype = sz
        lib.ssk_qssim_workspace_bytes.argtypes = [i32, i32, i32, i32, i32]
        lib.ssk_qssim.restype = i32
        lib.ssk_qssim.argtypes = [vp, vp, i32, i32, i32, i64, i64, i32, i32, ctypes.c_double, ctypes.c_double, vp,
                                  vp, sz, vp]
        lib.ssk_delta_e_workspace_bytes.restype = sz
        lib.ssk_delta_e_workspace_bytes.argtypes = [i32, i32, i32]
        lib.ssk_delta_e.restype = i32
        lib.ssk_delta_e.argtypes = [pC, pC, i32, i32, i32, i32, vp, i64, i64, vp, sz, vp]
        del pD
        lib.ssk_host_register.restype = i32
        lib.ssk_host_register.argtypes = [vp, sz, i32]
        lib.ssk_host_unregister.restype = i32
        lib.ssk_host_unregister.argtypes = [vp]
        lib.ssk_launch_count.restype = ctypes.c_uint64
        lib.ssk_probe_fp32_tflops.restype = i32
        lib.ssk_probe_fp32_tflops.argtypes = [ctypes.c_double, ctypes.POINTER(ctypes.c_double), vp]
        if lib.ssk_abi_version() != ABI_VERSION:
            raise EngineUnavailable("libssimk.so ABI version mismatch; rebuild it")
        _lib = lib
        return lib


def raise_for(rc: int, what: str = "") -> None:
    """Map a native return code onto the reference's exception classes."""
    if rc == 0:
        return
    msg = (_lib.ssk_strerror(rc).decode() if _lib is not None else str(rc)) + (f" ({what})" if what else "")
    if rc == E_WINDOW:
        raise WindowLargerThanImage(msg)
    if rc == E_LEVELS:
        raise TooManyLevels(msg)
    if rc == E_TOO_SMALL:
        raise TooSmall(msg)
    if rc in (E_ARG, E_SHAPE, E_ALIGN, E_WORKSPACE):
        raise ValidationError(msg)
    raise SsimkitError(msg)


# ---------------------------------------------------------------------------
# torch / device plumbing
# ---------------------------------------------------------------------------

_torch = None


def torch_mod():
    global _torch
    if _torch is None:
        import torch

        _torch = torch
    return _torch


def require_device():
    """The CUDA device the engine runs on; raises if there is none (no CPU fallback)."""
    torch = torch_mod()
    if not torch.cuda.is_available():
        raise EngineUnavailable("no CUDA device: the SSIM engine runs on a B200 only (no CPU fallback)")
    load_library()
    return torch.device("cuda", torch.cuda.current_device())


def lib() -> ctypes.CDLL:
    return load_library()


def stream_handle(stream=None) -> int:
    torch = torch_mod()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


_DT_CODES = None


def dtype_code(t) -> int:
    torch = torch_mod()
    global _DT_CODES
    if _DT_CODES is None:
        _DT_CODES = {torch.uint8: U8, torch.uint16: U16, torch.int16: U16, torch.uint32: U32,
                     torch.int32: U32, torch.float32: F32, torch.float64: F64}
    code = _DT_CODES.get(t.dtype)
    if code is None:
        raise ValidationError(f"unsupported device sample dtype {t.dtype}")
    return code


def esize(code: int) -> int:
    return {U8: 1, U16: 2, U32: 4, F32: 4, F64: 8}[code]


def aligned_pitch(w: int, code: int) -> int:
    es = esize(code)
    return ((w * es + 15) // 16) * 16 // es


def make_planes(ref, dist, code: int, bit_depth: int, scale_log2: int = 0) -> Planes:
    """Describe a [n, h, w] pair of CUDA tensors that share geometry and strides."""
    n, h, w = ref.shape
    return Planes(
        ref=ref.data_ptr(), dist=dist.data_ptr(), dtype=code, scale_log2=scale_log2,
        n=n, h=h, w=w, bit_depth=bit_depth, row_pitch=ref.stride(1), frame_pitch=ref.stride(0),
    )


def make_window(window, c1: float, c2: float) -> Window:
    """Window + constants.  Gaussian windows carry sigma; up to 31 taps also the taps
    g/sum(g) (float64, rounded to fp32) for the fp32 kernels, wider windows only sigma
    (the library builds fp64 taps for its generic kernel)."""
    win = Window(shape=GAUSS if window.shape == "gauss" else RECT, k=window.k, stride=window.stride,
                 _pad=0, c1=c1, c2=c2, sigma=0.0)
    if window.shape == "gauss":
        if window.k > GAUSS_MAX_K:
            raise ValidationError(f"gaussian windows wider than {GAUSS_MAX_K} taps are not supported")
        win.sigma = float(window.sigma)
        if window.k <= 31:
            for i, t in enumerate(gaussian_taps(window.sigma, window.k)):
                win.taps[i] = float(t)
    return win


def gaussian_taps(sigma: float, k: int) -> np.ndarray:
    """Normalised 1-D Gaussian: the separable factor of gaussian_kernel (src/stats.py:41-44)."""
    x = np.arange(k, dtype=np.float64) - (k - 1) / 2.0
    g = np.exp(-(x * x) / (2.0 * sigma * sigma))
    return g / g.sum()


class Workspace:
    """Grow-only device scratch per (device, stream) -- calls stay allocation-free."""

    def __init__(self):
        self._buf = {}
        self._lock = threading.Lock()

    def get(self, nbytes: int, device, stream=None):
        torch = torch_mod()
        key = (device.index, stream_handle(stream))
        with self._lock:
            buf = self._buf.get(key)
            if buf is None or buf.numel() < nbytes:
                buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
                self._buf[key] = buf
            return buf


WORKSPACE = Workspace()
