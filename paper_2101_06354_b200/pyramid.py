"""Multiscale SSIM over the dyadic pyramid (ssimkit src/multiscale.py) on the B200.

The whole pyramid runs on the device in one library call (``ssk_msssim``):
2x2 pyramid steps kept as exact scaled integers (each level-s sample is a sum
of 4^s input samples; the reference's float64 levels are exactly those values
times 4^-s, src/multiscale.py:19-33), then one fused SSIM pass per level that
reduces mean(cs) below the coarsest level and mean(l*cs) at it
(:50-58).  Only the per-level means come back; the exponent-weighted
combination is evaluated in float64 on the host exactly as the reference does
(:62-74).
"""

from __future__ import annotations

import numpy as np

from . import engine
from .errors import TooManyLevels, TooSmall, ValidationError
from .moments import check_fit, resolve_engine
from .options import MultiscaleSpec, SsimConfig
from .planes import LumaPlane, PlaneLike, plane_bit_depth, plane_data, validate_frame_pair


def dyadic_downsample(plane: PlaneLike) -> PlaneLike:
    """2x2 mean of the even-trimmed plane (src/multiscale.py:19-33), computed on the device."""
    a = plane_data(plane)
    h, w = a.shape
    if h < 2 or w < 2:
        raise TooSmall(f"cannot downsample a {w}x{h} plane")
    bd = plane_bit_depth(plane, 8)
    # integer planes stay exact scaled integers; float planes run in float64
    src = np.ascontiguousarray(a if a.dtype.kind in "ui" and a.min() >= 0 else a.astype(np.float64))
    pair = engine.upload_pair(src, src, bd, gauss=False)
    out = engine.downsample(pair)
    pooled = engine.to_float64(out.ref[0], out.code, out.scale_log2).cpu().numpy()
    if isinstance(plane, LumaPlane):
        return LumaPlane(pooled, plane.bit_depth)
    return pooled


def _check_levels(h: int, w: int, k: int, levels: int) -> None:
    if levels < 1:
        raise ValidationError("need at least one scale")
    if min(h, w) // (1 << (levels - 1)) < k:
        raise TooManyLevels(
            f"a {k}x{k} window does not fit the coarsest of {levels} scales of a {w}x{h} image"
        )


def _level_means(ref: PlaneLike, dist: PlaneLike, config: SsimConfig, levels: int) -> np.ndarray:
    a, b = plane_data(ref), plane_data(dist)
    h, w = a.shape
    _check_levels(h, w, config.window.k, levels)
    check_fit(h, w, config.window.k)
    resolve_engine(config.window, config.engine)
    bd = plane_bit_depth(ref, config.bit_depth)
    pair = engine.upload_pair(a, b, bd, config.window.shape == "gauss")
    means, _, _ = engine.msssim_levels(pair, config.window, config.c1, config.c2, levels)
    return means[0].cpu().numpy()


def scale_scores(ref: PlaneLike, dist: PlaneLike, config: SsimConfig, levels: int) -> list[float]:
    """Per-scale scores: mean cs at scales < L-1, mean l*cs at the coarsest (src/multiscale.py:36-59)."""
    return [float(x) for x in _level_means(ref, dist, config, levels)]


def combine_scale_scores(scores, spec: MultiscaleSpec) -> float:
    """Exponent-weighted product (negatives clamp to 0) or normalised sum (src/multiscale.py:62-74)."""
    exps = spec.effective_exponents()
    if len(scores) != len(exps):
        raise ValidationError(f"{len(scores)} scores for {len(exps)} exponents")
    if spec.aggregation == "sum":
        return float(sum(e * s for e, s in zip(exps, scores)))
    out = 1.0
    for e, s in zip(exps, scores):
        out *= max(s, 0.0) ** e
    return float(out)


def msssim(ref: PlaneLike, dist: PlaneLike, config: SsimConfig = SsimConfig(),
           spec: MultiscaleSpec | None = None) -> float:
    """Multiscale SSIM of a pair (src/multiscale.py:77-90)."""
    spec = MultiscaleSpec.product() if spec is None else spec
    if not spec.enabled:
        raise ValidationError("multiscale aggregation is off; use ssim_score instead")
    validate_frame_pair(ref, dist)
    return combine_scale_scores(scale_scores(ref, dist, config, spec.levels), spec)
