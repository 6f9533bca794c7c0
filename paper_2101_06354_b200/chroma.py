"""Channel-wise color SSIM (ssimkit src/color.py, cw/fixed models) on the B200.

Each channel is scored at its own resolution (4:2:0 chroma is not
upsampled, src/color.py:122-125, :144-153) by the fused SSIM kernel; only the
three per-channel means return to the host, where they are combined in
float64 with the reference's formulas.  The BT.709 conversions needed to
accept RGB input are plain per-pixel float64 maps kept here for API parity
(src/color.py:64-108); the quaternion / CIELAB / hue models are outside the
accelerated path.
"""

from __future__ import annotations

import numpy as np

from .errors import DegenerateWeights, ValidationError, WrongSpace
from .options import SsimConfig
from .planes import CHROMA_444, SPACE_RGB, SPACE_YCBCR, ColorFrame, LumaPlane, validate_color_pair
from .scoring import ssim_score

_KR, _KG, _KB = 0.213, 0.715, 0.072
_CB_SCALE, _CR_SCALE = 0.539, 0.635


def rgb_to_ycbcr_bt709(frame: ColorFrame) -> ColorFrame:
    """BT.709 RGB -> YCbCr, chroma offset by L/2 (src/color.py:64-73)."""
    frame.require_space(SPACE_RGB)
    r, g, b = (np.asarray(c, dtype=np.float64) for c in frame.channels)
    half = frame.peak / 2.0
    y = _KR * r + _KG * g + _KB * b
    return ColorFrame((y, _CB_SCALE * (b - y) + half, _CR_SCALE * (r - y) + half), SPACE_YCBCR,
                      frame.subsampling, frame.bit_depth)


def upsample_chroma(frame: ColorFrame) -> ColorFrame:
    """Nearest-neighbour 4:2:0 -> 4:4:4 (src/color.py:92-101)."""
    if frame.subsampling == CHROMA_444:
        return frame
    h, w = frame.height, frame.width
    up = [np.repeat(np.repeat(c, 2, axis=0), 2, axis=1)[:h, :w] for c in frame.channels[1:]]
    return ColorFrame((frame.channels[0], up[0], up[1]), frame.space, CHROMA_444, frame.bit_depth)


def ycbcr_bt709_to_rgb(frame: ColorFrame) -> ColorFrame:
    """Inverse BT.709 (4:4:4), clamped to the nominal range (src/color.py:76-89)."""
    frame.require_space(SPACE_YCBCR)
    frame = upsample_chroma(frame)
    y, cb, cr = (np.asarray(c, dtype=np.float64) for c in frame.channels)
    half = frame.peak / 2.0
    b = (cb - half) / _CB_SCALE + y
    r = (cr - half) / _CR_SCALE + y
    g = (y - _KR * r - _KB * b) / _KG
    return ColorFrame(tuple(np.clip(c, 0.0, frame.peak) for c in (r, g, b)), SPACE_RGB, CHROMA_444,
                      frame.bit_depth)


def luma_of(frame: ColorFrame) -> LumaPlane:
    """Luminance plane of an RGB or YCbCr frame (src/color.py:104-108)."""
    if frame.space == SPACE_YCBCR:
        return LumaPlane(frame.channels[0], frame.bit_depth)
    if frame.space == SPACE_RGB:
        r, g, b = (np.asarray(c, dtype=np.float64) for c in frame.channels)
        return LumaPlane(_KR * r + _KG * g + _KB * b, frame.bit_depth)
    raise WrongSpace(f"no luminance definition for {frame.space} frames")


def combine_channelwise(fy: float, fcb: float, fcr: float, alpha: float, beta: float) -> float:
    """(fY + alpha fCb + beta fCr) / (1 + alpha + beta) (src/color.py:111-116)."""
    denom = 1.0 + alpha + beta
    if abs(denom) < 1e-12:
        raise DegenerateWeights("1 + alpha + beta must be nonzero")
    return (fy + alpha * fcb + beta * fcr) / denom


def channel_scores(ref: ColorFrame, dist: ColorFrame, config: SsimConfig) -> tuple[float, float, float]:
    """Per-channel mean SSIM at each plane's own resolution (src/color.py:144-153)."""
    validate_color_pair(ref, dist)
    if ref.space == SPACE_RGB:
        ref, dist = rgb_to_ycbcr_bt709(ref), rgb_to_ycbcr_bt709(dist)
    elif ref.space != SPACE_YCBCR:
        raise WrongSpace(f"channel-wise scoring needs RGB or YCbCr frames, got {ref.space}")
    config = config.for_bit_depth(ref.bit_depth)
    return tuple(ssim_score(a, b, config) for a, b in zip(ref.channels, dist.channels))


def channelwise_cssim(ref: ColorFrame, dist: ColorFrame, alpha: float, beta: float,
                      config: SsimConfig = SsimConfig()) -> float:
    fy, fcb, fcr = channel_scores(ref, dist, config)
    return combine_channelwise(fy, fcb, fcr, alpha, beta)


def fixed_weight_cssim(ref: ColorFrame, dist: ColorFrame, weights=(0.8, 0.1, 0.1),
                       config: SsimConfig = SsimConfig()) -> float:
    """Convex channel combination (src/color.py:131-141)."""
    if abs(sum(weights) - 1.0) > 1e-9:
        raise ValidationError(f"channel weights must sum to 1, got {sum(weights)!r}")
    return float(sum(w * s for w, s in zip(weights, channel_scores(ref, dist, config))))
