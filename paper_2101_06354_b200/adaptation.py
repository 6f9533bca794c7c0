"""Resolution adaptation before scoring (ssimkit src/adaptation.py:23-110).

The scale factor a ``ScalePolicy`` prescribes is host arithmetic on the frame
geometry (legacy 256-line rule, its viewing-distance generalisation, SAST);
the resampler itself -- integer-factor block averaging with partial trailing
blocks -- runs on the device (``ssk_box_downsample``).  For integer samples
and a power-of-two factor that tiles the frame the downsampled plane stays an
exact scaled integer plane (block sums, value = sum * 2^-scale_log2), so the
rect/integral path downstream keeps its bit-exact integer arithmetic; other
cases produce the reference's float64 block means (one IEEE division of an
exact sum: bit-identical to ``box_downsample`` for integer samples).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _native as nat
from . import engine
from .errors import ValidationError
from .options import ScalePolicy
from .planes import LumaPlane, PlaneLike, plane_data


def round_half_away(x: float) -> int:
    """Nearest integer, halves away from zero (src/adaptation.py:23-25)."""
    mag = math.floor(abs(x) + 0.5)
    return int(mag) if x >= 0 else -int(mag)


def _rounded(ratio: float, rounding: str) -> int:
    return max(1, math.ceil(ratio) if rounding == "ceil" else round_half_away(ratio))


def legacy_scale_factor(width: int, height: int, rounding: str = "round") -> int:
    """The 256-line rule max(1, round(min(W, H) / 256)) (src/adaptation.py:28-34)."""
    if width <= 0 or height <= 0:
        raise ValidationError("dimensions must be positive")
    return _rounded(min(width, height) / 256.0, rounding)


def enhanced_scale_factor(width: int, height: int, d_over_h: float, rounding: str = "round") -> int:
    """256-line rule scaled by 3 / (D/H) (src/adaptation.py:37-47); D/H = 3 is the legacy rule."""
    if width <= 0 or height <= 0 or d_over_h <= 0:
        raise ValidationError("dimensions and d/h ratio must be positive")
    return _rounded((min(width, height) / 256.0) * (3.0 / d_over_h), rounding)


def viewing_geometry(display_height: float, distance: float, lines: int) -> tuple[float, float]:
    """(viewing angle in degrees, pixel-spacing frequency L / (2 alpha)) (src/adaptation.py:50-59)."""
    if display_height <= 0 or distance <= 0 or lines <= 0:
        raise ValidationError("geometry inputs must be positive")
    alpha = 2.0 * math.degrees(math.atan(display_height / (2.0 * distance)))
    return alpha, lines / (2.0 * alpha)


def sast_factor(display_height: float, display_width: float, distance: float,
                theta_h: float = 40.0, theta_w: float = 50.0) -> float:
    """Self-adaptive scale transform factor, >= 1 (src/adaptation.py:62-78)."""
    if min(display_height, display_width, distance, theta_h, theta_w) <= 0:
        raise ValidationError("geometry inputs must be positive")
    tan_prod = 4.0 * math.tan(math.radians(theta_h) / 2.0) * math.tan(math.radians(theta_w) / 2.0)
    z = math.sqrt((display_height / distance) * (display_width / distance) / tan_prod)
    return max(1.0, z)


def policy_factor(policy: ScalePolicy, width: int, height: int) -> int:
    """Integer downsampling factor of a policy for a W x H frame (src/adaptation.py:81-90)."""
    if policy.kind == "none":
        return 1
    if policy.kind == "legacy":
        return legacy_scale_factor(width, height, policy.rounding)
    if policy.kind == "dh":
        return enhanced_scale_factor(width, height, policy.d_over_h, policy.rounding)
    return max(1, round_half_away(sast_factor(height, width, policy.distance, policy.theta_h, policy.theta_w)))


def _check_factor(factor) -> None:
    if not isinstance(factor, int) or factor < 1:
        raise ValidationError(f"factor must be an integer >= 1, got {factor!r}")


def downsample_pair(pair: engine.DevicePair, factor: int, stream=None) -> engine.DevicePair:
    """Block-average both frames of a device batch by ``factor`` (one kernel launch)."""
    _check_factor(factor)
    if factor == 1:
        return pair
    torch = nat.torch_mod()
    n, h, w = pair.shape
    ho, wo = -(-h // factor), -(-w // factor)
    integer = pair.code in (nat.U8, nat.U16, nat.U32)
    pow2 = factor & (factor - 1) == 0
    top = float((1 << pair.bit_depth) - 1) * 2.0 ** pair.scale_log2 * factor * factor
    if integer and pow2 and h % factor == 0 and w % factor == 0 and top <= 4294967295.0:
        code = nat.U16 if top <= 65535.0 else nat.U32
        scale = pair.scale_log2 + 2 * (factor.bit_length() - 1)
    else:
        code, scale = nat.F64, 0
    t_dt = {nat.U16: torch.uint16, nat.U32: torch.uint32, nat.F64: torch.float64}[code]
    pitch = nat.aligned_pitch(wo, code)
    buf = torch.empty((2, n, ho, pitch), dtype=t_dt, device=pair.ref.device)
    rc = nat.lib().ssk_box_downsample(ctypes.byref(pair.planes()), factor, buf[0].data_ptr(), buf[1].data_ptr(),
                                      code, pitch, ho * pitch, nat.stream_handle(stream))
    nat.raise_for(rc, "box downsample")
    return engine.DevicePair(buf[0, :, :, :wo], buf[1, :, :, :wo], code, pair.bit_depth, scale)


def box_downsample(plane: PlaneLike, factor: int) -> PlaneLike:
    """Block means by an integer factor, float64 out (src/adaptation.py:93-110), on the device."""
    _check_factor(factor)
    if factor == 1:
        return plane
    arr = np.asarray(plane_data(plane))
    if arr.ndim != 2 or arr.size == 0:
        raise ValidationError("box_downsample takes a non-empty 2-D plane")
    bd = plane.bit_depth if isinstance(plane, LumaPlane) else 8
    pair = engine.upload_pair(arr, arr, bd, gauss=False)
    out = downsample_pair(pair, factor)
    vals = engine.to_float64(out.ref, out.code, out.scale_log2)[0].cpu().numpy()
    if isinstance(plane, LumaPlane):
        return LumaPlane(vals, plane.bit_depth)
    return vals


def scale_frame(frame, factor: int):
    """``_scale_frame`` (src/pipeline.py:172-178): luma planes and every channel of a color frame."""
    if factor == 1:
        return frame
    from .planes import ColorFrame

    if isinstance(frame, ColorFrame):
        return ColorFrame(tuple(box_downsample(c, factor) for c in frame.channels), frame.space,
                          frame.subsampling, frame.bit_depth)
    return box_downsample(frame, factor)

