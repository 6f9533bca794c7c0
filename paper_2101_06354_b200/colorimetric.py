"""Colorimetric similarity models on the B200 (ssimkit src/color.py:159-371).

* ``qssim``  -- quaternion SSIM: channels embedded as pure quaternions (RGB,
  BT.709 YCbCr or scaled CIELAB), twelve windowed means per window in one
  kernel (``ssk_qssim``), each accumulated in the reference's (m, n) order.
* ``cmssim`` -- luma SSIM map weighted by clamp(1 - dE/45, 0, 1), dE the
  CIELAB difference after opponent-space chroma smoothing, sampled at the
  window centres (``ssk_delta_e``) and applied by the device pooler.
* ``hssim``  -- (luma SSIM + 0.2 * hue-plane SSIM) / 1.2 on the fused SSIM
  kernels.

Frames are uploaded once; every conversion (BT.709 in both directions with
4:2:0 nearest upsampling, luma, HSV hue, CIELAB) is a device kernel
(``ssk_color_convert``) and only scalars (or the maps the reference API
returns) come back.  Per-pair signatures and return types follow the
reference; batching frames is a matter of n > 1 in the C ABI.
"""

from __future__ import annotations

import ctypes
from dataclasses import replace

import numpy as np

from . import _native as nat
from . import engine
from .errors import ValidationError, WrongSpace
from .options import SsimConfig, WindowSpec
from .planes import CHROMA_420, SPACE_RGB, SPACE_YCBCR, ColorFrame, LumaPlane, validate_color_pair


class DeviceColor:
    """One color frame resident in HBM (three planes + the ``ssk_color`` descriptor)."""

    def __init__(self, planes, code: int, space: int, sub420: bool, h: int, w: int, bit_depth: int):
        self.planes = planes  # three [1, h_c, w_c] tensors (kept alive for the descriptor)
        self.code, self.space, self.sub420 = code, space, sub420
        self.h, self.w, self.bit_depth = h, w, bit_depth
        self.peak = float((1 << bit_depth) - 1)
        c = nat.Color()
        for i, t in enumerate(planes):
            c.ch[i] = t.data_ptr()
            c.row_pitch[i] = t.stride(1)
            c.frame_pitch[i] = t.stride(0)
        c.dtype, c.space, c.subsampling = code, space, int(sub420)
        c.n, c.h, c.w, c.bit_depth = 1, h, w, bit_depth
        self.desc = c

    @classmethod
    def from_frame(cls, frame: ColorFrame) -> "DeviceColor":
        torch = nat.torch_mod()
        dev = nat.require_device()
        if frame.space == SPACE_RGB:
            space = nat.SPACE_RGB
        elif frame.space == SPACE_YCBCR:
            space = nat.SPACE_YCBCR
        else:
            raise WrongSpace(f"color models take RGB or BT.709 YCbCr frames, got {frame.space}")
        chans = [np.asarray(c) for c in frame.channels]
        if all(c.dtype == np.uint8 for c in chans):
            code, dt = nat.U8, np.uint8
        elif all(c.dtype.kind in "ui" for c in chans) and max(int(c.max()) for c in chans) <= 0xFFFF \
                and min(int(c.min()) for c in chans) >= 0:
            code, dt = nat.U16, np.uint16
        else:
            code, dt = nat.F64, np.float64
        planes = [torch.from_numpy(np.array(c, dtype=dt, order="C")).to(dev).unsqueeze(0) for c in chans]
        return cls(planes, code, space, frame.subsampling == CHROMA_420, frame.height, frame.width, frame.bit_depth)

    def convert(self, op: int, stream=None):
        """[planes, h, w] float64 device tensor of a conversion (``ssk_color_convert``)."""
        torch = nat.torch_mod()
        nplanes = 1 if op in (nat.CONV_LUMA, nat.CONV_HUE) else 3
        out = torch.empty((nplanes, self.h, self.w), dtype=torch.float64, device=self.planes[0].device)
        rc = nat.lib().ssk_color_convert(ctypes.byref(self.desc), op, out.data_ptr(), self.w,
                                         nplanes * self.h * self.w, nat.stream_handle(stream))
        nat.raise_for(rc, "color conversion")
        return out

    def as_rgb(self) -> "DeviceColor":
        """RGB float64 planes (ycbcr_bt709_to_rgb for YCbCr frames, src/color.py:76-89)."""
        if self.space == nat.SPACE_RGB:
            return self
        rgb = self.convert(nat.CONV_RGB)
        return DeviceColor([rgb[i:i + 1] for i in range(3)], nat.F64, nat.SPACE_RGB, False, self.h, self.w,
                           self.bit_depth)

    def require_rgb(self) -> "DeviceColor":
        if self.space != nat.SPACE_RGB:
            raise WrongSpace(f"expected a {SPACE_RGB} frame, got {SPACE_YCBCR}")
        return self


def _device_pair(ref: ColorFrame, dist: ColorFrame) -> tuple[DeviceColor, DeviceColor]:
    validate_color_pair(ref, dist)
    return DeviceColor.from_frame(ref), DeviceColor.from_frame(dist)


def _host_frame(planes, space: str, bit_depth: int) -> ColorFrame:
    chans = tuple(planes[i].cpu().numpy() for i in range(3))
    return ColorFrame(chans, space, "444", bit_depth)


# ---------------------------------------------------------------------------
# conversions with the reference's signatures (src/color.py:64-108, :341-362)
# ---------------------------------------------------------------------------

def rgb_to_ycbcr_bt709(frame: ColorFrame) -> ColorFrame:
    frame.require_space(SPACE_RGB)
    if frame.subsampling == CHROMA_420:
        raise ValidationError("RGB frames are 4:4:4")
    return _host_frame(DeviceColor.from_frame(frame).convert(nat.CONV_YCBCR), SPACE_YCBCR, frame.bit_depth)


def ycbcr_bt709_to_rgb(frame: ColorFrame) -> ColorFrame:
    frame.require_space(SPACE_YCBCR)
    return _host_frame(DeviceColor.from_frame(frame).convert(nat.CONV_RGB), SPACE_RGB, frame.bit_depth)


def luma_of(frame: ColorFrame) -> LumaPlane:
    if frame.space == SPACE_YCBCR:
        return LumaPlane(frame.channels[0], frame.bit_depth)
    if frame.space != SPACE_RGB:
        raise WrongSpace(f"no luminance definition for {frame.space} frames")
    y = DeviceColor.from_frame(frame).convert(nat.CONV_LUMA)[0].cpu().numpy()
    return LumaPlane(y, frame.bit_depth)


def hue_plane(frame: ColorFrame) -> LumaPlane:
    """HSV hue rescaled to [0, L]; achromatic pixels 0 (src/color.py:341-362)."""
    frame.require_space(SPACE_RGB)
    hue = DeviceColor.from_frame(frame).convert(nat.CONV_HUE)[0].cpu().numpy()
    return LumaPlane(hue, frame.bit_depth)


# ---------------------------------------------------------------------------
# models
# ---------------------------------------------------------------------------

def _embedding(dc: DeviceColor, space: str):
    """qssim's embedding channels (src/color.py:159-178) as [3, h, w] float64."""
    if space == "rgb":
        return dc.require_rgb().convert(nat.CONV_RGB)
    if space == "ycbcr":
        return dc.convert(nat.CONV_YCBCR)
    if space == "lab":
        return dc.require_rgb().convert(nat.CONV_LAB_EMBED)
    raise ValidationError(f"unknown quaternion embedding space {space!r}")


def qssim(ref: ColorFrame, dist: ColorFrame, window: WindowSpec = WindowSpec.rectangular(11), k1: float = 0.01,
          k2: float = 0.03, space: str = "rgb") -> float:
    """Quaternion color similarity, windowed and averaged (src/color.py:181-256)."""
    validate_color_pair(ref, dist)
    if window.shape != "rect":
        raise ValidationError("quaternion similarity uses rectangular windows")
    k, stride = window.k, window.stride
    if k > ref.height or k > ref.width:
        raise ValidationError(f"{k}x{k} window does not fit a {ref.width}x{ref.height} frame")
    a, b = _device_pair(ref, dist)
    e1, e2 = _embedding(a, space), _embedding(b, space)
    peak = ref.peak
    torch = nat.torch_mod()
    h, w = ref.height, ref.width
    lib = nat.lib()
    ws_bytes = lib.ssk_qssim_workspace_bytes(1, h, w, k, stride)
    ws = nat.WORKSPACE.get(max(ws_bytes, 256), e1.device)
    out = torch.empty((1,), dtype=torch.float64, device=e1.device)
    rc = lib.ssk_qssim(e1.data_ptr(), e2.data_ptr(), 1, h, w, w, 3 * h * w, k, stride, (k1 * peak) ** 2,
                       (k2 * peak) ** 2, out.data_ptr(), ws.data_ptr(), ws.numel(), nat.stream_handle())
    nat.raise_for(rc, "qssim")
    return float(out[0].item())


def _delta_e_grid(a: DeviceColor, b: DeviceColor, k: int, stride: int, mode: int, smooth: bool = True):
    torch = nat.torch_mod()
    gh, gw = (a.h - k) // stride + 1, (a.w - k) // stride + 1
    out = torch.empty((1, gh, gw), dtype=torch.float64, device=a.planes[0].device)
    lib = nat.lib()
    ws_bytes = lib.ssk_delta_e_workspace_bytes(1, a.h, a.w)
    ws = nat.WORKSPACE.get(max(ws_bytes, 256), out.device)
    rc = lib.ssk_delta_e(ctypes.byref(a.desc), ctypes.byref(b.desc), int(smooth), k, stride, mode, out.data_ptr(),
                         gw, gh * gw, ws.data_ptr(), ws.numel(), nat.stream_handle())
    nat.raise_for(rc, "delta E")
    return out


def delta_e_map(ref: ColorFrame, dist: ColorFrame, smooth_opponent: bool = True) -> np.ndarray:
    """Per-pixel CIELAB distance after the opponent-space chroma smoothing (src/color.py:290-296)."""
    validate_color_pair(ref, dist)
    ref.require_space(SPACE_RGB)
    dist.require_space(SPACE_RGB)
    a, b = _device_pair(ref, dist)
    return _delta_e_grid(a, b, 1, 1, 0, smooth_opponent)[0].cpu().numpy()


def _plane_ssim(p1, p2, config: SsimConfig, want: int):
    """Fused SSIM of two [1, h, w] float64 device planes; returns (sums, maps, count)."""
    win = config.window
    pair = engine.device_pair(p1, p2, config.bit_depth, win.shape == "gauss")
    _, h, w = pair.shape
    from .moments import check_fit, resolve_engine

    check_fit(h, w, win.k)
    resolve_engine(win, config.engine)
    sums, maps = engine.ssim(pair, win, config.c1, config.c2, want)
    gh, gw = engine.grid_shape(h, w, win.k, win.stride)
    return sums, maps, gh * gw


def _rgb_models_pair(ref: ColorFrame, dist: ColorFrame, window: WindowSpec, config: SsimConfig):
    validate_color_pair(ref, dist)
    a, b = _device_pair(ref, dist)
    a, b = a.as_rgb(), b.as_rgb()
    config = config.for_bit_depth(ref.bit_depth)
    if config.window != window:
        config = replace(config, window=window)
    return a, b, config


def cmssim(ref: ColorFrame, dist: ColorFrame, window: WindowSpec = WindowSpec.rectangular(11),
           config: SsimConfig = SsimConfig()) -> float:
    """Luma SSIM map weighted down by the CIELAB difference (src/color.py:299-334)."""
    from .pooling import pool_maps

    a, b, config = _rgb_models_pair(ref, dist, window, config)
    _, maps, _ = _plane_ssim(a.convert(nat.CONV_LUMA), b.convert(nat.CONV_LUMA), config,
                             nat.WANT_Q | nat.MAP_TERMS)
    weights = _delta_e_grid(a, b, window.k, window.stride, 1)
    # lw pooling with a = 0, b = 1 applies clip(w, 0, 1) * q and averages
    pooled, _ = pool_maps(maps[:, 2].double(), "lw:a=0,b=1", weights)
    return float(pooled[0].item())


def hssim(ref: ColorFrame, dist: ColorFrame, window: WindowSpec = WindowSpec.rectangular(11),
          config: SsimConfig = SsimConfig()) -> float:
    """(SSIM + 0.2 * hue-channel SSIM) / 1.2 (src/color.py:365-371)."""
    a, b, config = _rgb_models_pair(ref, dist, window, config)
    sl, _, n = _plane_ssim(a.convert(nat.CONV_LUMA), b.convert(nat.CONV_LUMA), config, nat.WANT_Q)
    sh, _, _ = _plane_ssim(a.convert(nat.CONV_HUE), b.convert(nat.CONV_HUE), config, nat.WANT_Q)
    means = engine.frame_means(nat.torch_mod().stack([sl[0, 0], sh[0, 0]]), n).cpu().numpy()
    luma_score, hue_score = float(means[0]), float(means[1])
    return (luma_score + 0.2 * hue_score) / 1.2
