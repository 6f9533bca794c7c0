"""Channel-wise color SSIM (ssimkit src/color.py, cw/fixed models) on the B200.

Each channel is scored at its own resolution (4:2:0 chroma is not
upsampled, src/color.py:122-125, :144-153) as the reference defines it,
mssim(ssim_map(..)): the map stays on the device and its mean is taken in
numpy's pairwise order; only the three per-channel means return to the host,
where they are combined in float64 with the reference's formulas.  (The
throughput path, ``batch.color_batch``, uses the fused score kernels.)  The BT.709 conversions needed to
accept RGB input run on the device (``colorimetric.py``, src/color.py:64-108),
as do the quaternion / CIELAB / hue models.
"""

from __future__ import annotations

import numpy as np

from .errors import DegenerateWeights, ValidationError, WrongSpace
from .options import SsimConfig
from .planes import CHROMA_444, SPACE_RGB, SPACE_YCBCR, ColorFrame, validate_color_pair
from .scoring import map_mean_score

from .colorimetric import luma_of, rgb_to_ycbcr_bt709, ycbcr_bt709_to_rgb  # noqa: F401  (device conversions)


def upsample_chroma(frame: ColorFrame) -> ColorFrame:
    """Nearest-neighbour 4:2:0 -> 4:4:4 (src/color.py:92-101): pure sample replication."""
    if frame.subsampling == CHROMA_444:
        return frame
    h, w = frame.height, frame.width
    up = [np.repeat(np.repeat(c, 2, axis=0), 2, axis=1)[:h, :w] for c in frame.channels[1:]]
    return ColorFrame((frame.channels[0], up[0], up[1]), frame.space, CHROMA_444, frame.bit_depth)


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
    # the reference's own definition, mssim(ssim_map(..)) per plane: the map on the device
    # (fp64 for Gaussian windows, exact for rect) and its numpy-order mean (ssk_pairwise_sum)
    return tuple(map_mean_score(a, b, config) for a, b in zip(ref.channels, dist.channels))


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
