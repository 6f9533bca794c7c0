"""Windowed local statistics (ssimkit src/stats.py), computed on the B200.

Public names and semantics follow the reference: valid-region windows
anchored at (0, 0) on the stride grid, Gaussian windows with normalised
weights (area 1), rect windows with area k^2, variances clamped at 0 and
covariance unclamped (src/stats.py:185-202), ``engine`` resolution
auto -> integral for rect / naive for Gaussian (:223-228).

On the device both rect engines are one kernel family: integer samples give
exact integer window sums either way (the reference's int64 integral tables
and its float64 direct sums agree exactly on integer input), so
``engine`` only selects validation behaviour here.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from . import engine
from .errors import EngineShapeMismatch, NonPositiveSigma, ValidationError, WindowLargerThanImage, WindowOutOfBounds
from .options import WindowSpec, default_gaussian_size
from .planes import PlaneLike, plane_bit_depth, plane_data, validate_frame_pair

TABLE_IDS = ("sum1", "sum2", "sq1", "sq2", "prod")


def gaussian_kernel(sigma: float, k: int | None = None) -> np.ndarray:
    """Normalised 2-D Gaussian weights (host float64, src/stats.py:30-44)."""
    if sigma <= 0:
        raise NonPositiveSigma(f"sigma must be positive, got {sigma}")
    k = default_gaussian_size(sigma) if k is None else k
    if k < 1:
        raise ValidationError(f"kernel size must be >= 1, got {k}")
    c = np.arange(k, dtype=np.float64) - (k - 1) / 2.0
    g = np.exp(-(c * c) / (2.0 * sigma * sigma))
    full = np.outer(g, g)
    return full / full.sum()


def rect_equivalent(sigma: float, mode: str) -> int:
    """Rect window size matching a Gaussian (src/stats.py:47-63)."""
    if sigma <= 0:
        raise NonPositiveSigma(f"sigma must be positive, got {sigma}")
    half = {"same-variance": lambda: math.ceil(sigma * math.sqrt(3.0)),
            "same-bandwidth": lambda: math.ceil(1.602 * sigma)}
    if mode == "same-size":
        return default_gaussian_size(sigma)
    if mode not in half:
        raise ValidationError(f"unknown equivalence mode {mode!r}")
    return 2 * half[mode]() + 1


@dataclass(frozen=True)
class IntegralSet:
    """Five summed-area tables with a zero border (int64 for integer samples)."""

    sum1: np.ndarray
    sum2: np.ndarray
    sq1: np.ndarray
    sq2: np.ndarray
    prod: np.ndarray
    height: int
    width: int

    def table(self, which: str) -> np.ndarray:
        if which not in TABLE_IDS:
            raise ValidationError(f"unknown table {which!r}, expected one of {TABLE_IDS}")
        return getattr(self, which)


def _gauss_like(window) -> bool:
    return window is not None and window.shape == "gauss"


def _pair_to_device(ref: PlaneLike, dist: PlaneLike, bit_depth: int, gauss: bool):
    a, b = plane_data(ref), plane_data(dist)
    return engine.upload_pair(a, b, bit_depth, gauss, validated=True)  # callers validated the pair


def build_integral_set(ref: PlaneLike, dist: PlaneLike) -> IntegralSet:
    """The five SATs of a validated pair, built on the device (src/stats.py:96-116)."""
    ref, dist = validate_frame_pair(ref, dist)
    bd = plane_bit_depth(ref, 8)
    a, b = plane_data(ref), plane_data(dist)
    both_int = a.dtype.kind in "uib" and b.dtype.kind in "uib"
    pair = engine.upload_pair(a, b, bd, gauss=False, validated=True)
    if both_int and pair.code not in (nat.U8, nat.U16):
        raise ValidationError("integer samples beyond 16 bits are not supported by the integral engine")
    if not both_int and pair.code != nat.F64:
        pair = engine.DevicePair(pair.ref.double(), pair.dist.double(), nat.F64, pair.bit_depth)
    t = engine.integral_tables(pair)[0].cpu().numpy()
    h, w = a.shape
    return IntegralSet(*(t[i] for i in range(5)), height=h, width=w)


def window_sum(iset: IntegralSet, which: str, i: int, j: int, k: int):
    """One k x k window sum from a table by the four-corner rule (src/stats.py:119-127)."""
    t = iset.table(which)
    if k < 1 or i < 0 or j < 0 or i + k > iset.height or j + k > iset.width:
        raise WindowOutOfBounds(
            f"{k}x{k} window at ({i}, {j}) leaves the {iset.width}x{iset.height} valid region"
        )
    return (t[i + k, j + k] + t[i, j] - t[i + k, j] - t[i, j + k]).item()


@dataclass(frozen=True)
class LocalStatsMaps:
    """mu1, mu2, var1, var2, cov on the window grid (src/stats.py:167-182)."""

    mu1: np.ndarray
    mu2: np.ndarray
    var1: np.ndarray
    var2: np.ndarray
    cov: np.ndarray
    window_size: int
    stride: int
    source_dims: tuple

    @property
    def grid_shape(self) -> tuple:
        return self.mu1.shape


def resolve_engine(window: WindowSpec, engine_name: str) -> str:
    """auto -> integral (rect) / naive (gauss); integral+gauss is an error (src/stats.py:223-228)."""
    if engine_name == "auto":
        engine_name = "integral" if window.shape == "rect" else "naive"
    if engine_name not in ("naive", "integral"):
        raise ValidationError(f"unknown engine {engine_name!r}")
    if engine_name == "integral" and window.shape != "rect":
        raise EngineShapeMismatch("the integral engine supports rectangular windows only")
    return engine_name


def check_fit(h: int, w: int, k: int) -> None:
    if k > h or k > w:
        raise WindowLargerThanImage(f"{k}x{k} window does not fit a {w}x{h} image")


def local_statistics(ref: PlaneLike, dist: PlaneLike, window: WindowSpec, engine: str = "auto") -> LocalStatsMaps:
    """Local moments of a pair on the device; float64 host arrays out."""
    ref, dist = validate_frame_pair(ref, dist)
    h, w = plane_data(ref).shape
    check_fit(h, w, window.k)
    resolve_engine(window, engine)
    bd = plane_bit_depth(ref, 8)
    pair = _pair_to_device(ref, dist, bd, _gauss_like(window))
    peak = float((1 << bd) - 1)
    _, maps = engine_ssim(pair, window, (0.01 * peak) ** 2, (0.03 * peak) ** 2, nat.MAP_STATS | nat.MAP_F64)
    m = maps[0].double().cpu().numpy()
    return LocalStatsMaps(mu1=m[0], mu2=m[1], var1=m[2], var2=m[3], cov=m[4], window_size=window.k,
                          stride=window.stride, source_dims=(h, w))


def engine_ssim(pair, window, c1, c2, want):
    return engine.ssim(pair, window, c1, c2, want)


def stats_from_sums(s1, s2, q1, q2, p12, area: float):
    """Moments from raw window sums over ``area`` samples (src/stats.py:185-202): the fp64
    elementwise kernel ``ssk_stats_from_sums`` (the reference's operation order, bit-identical)."""
    torch = nat.torch_mod()
    dev = nat.require_device()
    arrs = [np.asarray(x, dtype=np.float64) for x in (s1, s2, q1, q2, p12)]
    shape = np.broadcast_shapes(*(a.shape for a in arrs))
    if not float(area) > 0.0:
        raise ValidationError(f"window area must be positive, got {area!r}")
    if int(np.prod(shape)) == 0:
        return tuple(np.zeros(shape) for _ in range(5))
    t = torch.from_numpy(np.stack([np.broadcast_to(a, shape).ravel() for a in arrs])).to(dev)
    out = torch.empty((5, t.shape[1]), dtype=torch.float64, device=dev)
    nat.raise_for(nat.lib().ssk_stats_from_sums(*(t[i].data_ptr() for i in range(5)), t.shape[1], float(area),
                                                 out.data_ptr(), nat.stream_handle(None)), "stats_from_sums")
    host = out.cpu().numpy()
    return tuple(host[i].reshape(shape) for i in range(5))
