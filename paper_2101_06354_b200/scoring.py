"""SSIM term maps and pooled scores (ssimkit src/ssim.py) on the B200.

``ssim_map`` returns the reference's container types (``SsimTermMaps`` of
float64 ``QualityMap``) and therefore ends in a device->host copy; the
throughput entry points (``ssim_score`` here, ``batch.ssim_batch``) never
materialise a map: the fused kernel reduces sum(q) (and sum(l), sum(cs)) per
frame in its epilogue and only 24 bytes per frame leave the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Union

import numpy as np

from . import _native as nat
from . import engine
from .errors import EmptyMap
from .moments import LocalStatsMaps, check_fit, resolve_engine
from .options import SsimConfig
from .planes import PlaneLike, QualityMap, plane_bit_depth, plane_data, validate_frame_pair


@dataclass(frozen=True)
class SsimTermMaps:
    """Luminance, contrast-structure and combined quality maps (src/ssim.py:22-28)."""

    l_map: QualityMap
    cs_map: QualityMap
    q_map: QualityMap


def _prepare(ref: PlaneLike, dist: PlaneLike, config: SsimConfig):
    ref, dist = validate_frame_pair(ref, dist)
    a, b = plane_data(ref), plane_data(dist)
    h, w = a.shape
    check_fit(h, w, config.window.k)
    resolve_engine(config.window, config.engine)
    pair = engine.upload_pair(a, b, plane_bit_depth(ref, config.bit_depth), config.window.shape == "gauss",
                              validated=True)
    return pair, (h, w)


def term_maps_from_stats(stats: LocalStatsMaps, c1: float, c2: float) -> SsimTermMaps:
    """l, cs, q from given statistics grids (src/ssim.py:31-46): the fp64 elementwise kernel
    ``ssk_term_maps`` (the reference's operation order, bit-identical)."""
    torch = nat.torch_mod()
    dev = nat.require_device()
    grids = [np.asarray(x, dtype=np.float64) for x in (stats.mu1, stats.mu2, stats.var1, stats.var2, stats.cov)]
    shape = grids[0].shape
    geom = dict(stride=stats.stride, source_dims=stats.source_dims)
    if grids[0].size == 0:
        return SsimTermMaps(*(QualityMap(np.zeros(shape), **geom) for _ in range(3)))
    t = torch.from_numpy(np.stack([g.ravel() for g in grids])).to(dev)
    out = torch.empty((3, t.shape[1]), dtype=torch.float64, device=dev)
    nat.raise_for(nat.lib().ssk_term_maps(*(t[i].data_ptr() for i in range(5)), t.shape[1], float(c1), float(c2),
                                           out.data_ptr(), nat.stream_handle(None)), "term_maps_from_stats")
    host = out.cpu().numpy()
    return SsimTermMaps(*(QualityMap(host[i].reshape(shape), **geom) for i in range(3)))


def ssim_map(ref: PlaneLike, dist: PlaneLike, config: SsimConfig = SsimConfig()) -> SsimTermMaps:
    """SSIM term maps of a pair (src/ssim.py:49-52)."""
    pair, dims = _prepare(ref, dist, config)
    # Gaussian maps from the fp64 kernel (the reference's precision); rect maps are exact anyway
    _, maps = engine.ssim(pair, config.window, config.c1, config.c2,
                          nat.WANT_Q | nat.WANT_L | nat.WANT_CS | nat.MAP_TERMS | nat.MAP_F64)
    m = maps[0].double().cpu().numpy()
    geom = dict(stride=config.window.stride, source_dims=dims)
    return SsimTermMaps(QualityMap(m[0], **geom), QualityMap(m[1], **geom), QualityMap(m[2], **geom))


def mssim(maps: Union[SsimTermMaps, QualityMap, np.ndarray]) -> float:
    """Mean of a quality map (src/ssim.py:55-65), pooled on the device ('am' pooler).

    The throughput path never materialises maps (``ssim_score`` pools inside the
    SSIM kernel); this is the reference's map-level entry point."""
    from .pooling import pool_spatial

    if isinstance(maps, SsimTermMaps):
        v = maps.q_map.values
    elif isinstance(maps, QualityMap):
        v = maps.values
    else:
        v = np.asarray(maps, dtype=np.float64)
    if v.size == 0:
        raise EmptyMap("cannot average an empty quality map")
    return pool_spatial(v, "am")


def map_mean_score(ref: PlaneLike, dist: PlaneLike, config: SsimConfig = SsimConfig()) -> float:
    """mssim(ssim_map(ref, dist, config)) without the map leaving the device: the q map
    (fp64 for Gaussian windows) and its numpy-order mean (``ssk_pairwise_sum``), i.e. the
    reference's definition of a plane's score, bit for bit where the maps are."""
    from .pooling import SpatialPooler, _pool_exact

    pair, _ = _prepare(ref, dist, config)
    _, maps = engine.ssim(pair, config.window, config.c1, config.c2, nat.WANT_Q | nat.MAP_TERMS | nat.MAP_F64)
    return _pool_exact(maps[0, 2], SpatialPooler("am"))


def ssim_terms(ref: PlaneLike, dist: PlaneLike, config: SsimConfig = SsimConfig()) -> tuple[float, float, float]:
    """(mean q, mean l, mean cs) of a pair from one fused pass; no map leaves the GPU."""
    pair, (h, w) = _prepare(ref, dist, config)
    sums, _ = engine.ssim(pair, config.window, config.c1, config.c2, nat.WANT_Q | nat.WANT_L | nat.WANT_CS)
    gh, gw = engine.grid_shape(h, w, config.window.k, config.window.stride)
    s = engine.frame_means(sums, gh * gw)[0].cpu().numpy()
    return float(s[0]), float(s[1]), float(s[2])


def ssim_score(ref: PlaneLike, dist: PlaneLike, config: SsimConfig = SsimConfig()) -> float:
    """Mean SSIM of a pair (src/ssim.py:68-70) via the fused score-only kernel."""
    return ssim_terms(ref, dist, config)[0]


def weber_luminance_term(mu1: float, luminance_shift: float, c1_over_mu1sq: float) -> float:
    """Closed-form luminance term under mu2 = mu1 (1 + shift) (src/ssim.py:73-86)."""
    if mu1 <= 0:
        raise ValueError(f"mu1 must be positive, got {mu1}")
    r = 1.0 + luminance_shift
    return (2.0 * r + c1_over_mu1sq) / (1.0 + r ** 2 + c1_over_mu1sq)


def weber_contrast_term(contrast_shift: float, c2_over_var1: float) -> float:
    """Contrast-masking analogue under sigma2 = (1 + shift) sigma1 (src/ssim.py:89-92)."""
    r = 1.0 + contrast_shift
    return (2.0 * r + c2_over_var1) / (1.0 + r ** 2 + c2_over_var1)
