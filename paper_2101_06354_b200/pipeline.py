"""Per-frame scoring contract and presets of the reference pipeline (src/pipeline.py).

``luma_records`` is the device core every luma path funnels into: resolution
adaptation (``ssk_box_downsample``), then either the MS-SSIM pyramid call or
the fused SSIM pass, then spatial pooling -- mean pooling fused into the SSIM
kernel's reduction, any other pooler on the device over the q map the same
pass wrote (``ssk_pool_spatial``).  Results are per-frame float64 device
tensors for a whole batch, so the ``enhanced`` preset (rect 11 stride 5,
integral engine, dh:3 box downsampling, CoV pooling; src/pipeline.py:89-97)
runs as a handful of launches per batch with only scalars leaving the GPU.

``score_frame_pair`` keeps the reference's single-pair signature and record
(src/pipeline.py:189-258); ``PipelineSpec`` / ``preset_specs`` /
``expand_preset`` mirror :66-112.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional

from . import _native as nat
from . import engine
from .adaptation import downsample_pair, policy_factor, scale_frame
from .errors import DimensionMismatch, TooManyLevels, ValidationError
from .moments import check_fit, resolve_engine
from .options import ColorModelSpec, ScalePolicy, SsimConfig, WindowSpec
from .pooling import parse_spatial, pool_maps

#: Per-frame record schema, in report column order (src/pipeline.py:57-58).
FRAME_FIELDS = ("frame", "score", "am", "l_mean", "cs_mean")


@dataclass
class FrameScore:
    score: float
    am: Optional[float]
    l_mean: Optional[float]
    cs_mean: Optional[float]


@dataclass
class FrameRecords:
    """Per-frame fields of a batch as [n] float64 device tensors (None where the
    reference record has None: multiscale and color models report the score only)."""

    score: "object"
    am: "object" = None
    l_mean: "object" = None
    cs_mean: "object" = None

    def host(self, i: int) -> FrameScore:
        def f(t):
            return None if t is None else float(t[i])

        return FrameScore(f(self.score), f(self.am), f(self.l_mean), f(self.cs_mean))


@dataclass(frozen=True)
class PipelineSpec:
    """A resolved scoring pipeline: config + temporal depth + report format (src/pipeline.py:66-86)."""

    config: SsimConfig = field(default_factory=SsimConfig)
    kt: int = 1
    report_format: str = "jsonl"
    preset: Optional[str] = None
    workers: int = 1

    def __post_init__(self):
        if self.report_format not in ("jsonl", "csv"):
            raise ValidationError(f"unknown report format {self.report_format!r}")
        if not isinstance(self.kt, int) or isinstance(self.kt, bool) or self.kt < 1:
            raise ValidationError("kt must be an integer >= 1")
        if self.kt > 1 and self.config.color.model != "luma":
            raise ValidationError("spatio-temporal scoring operates on the luminance channel only")
        if self.kt > 1 and self.config.window.shape != "rect":
            raise ValidationError("spatio-temporal scoring needs a rectangular window")
        if not isinstance(self.workers, int) or self.workers < 1:
            raise ValidationError("workers must be an integer >= 1")


def enhanced_config() -> SsimConfig:
    """The ``enhanced`` preset's configuration (src/pipeline.py:89-97)."""
    return SsimConfig(window=WindowSpec.rectangular(11, stride=5), engine="integral",
                      scaling=ScalePolicy.enhanced_dh(3.0), color=ColorModelSpec.luma(),
                      spatial_pool="cov", temporal_pool="am")


def preset_specs() -> dict:
    return {"default": PipelineSpec(SsimConfig(), preset="default"),
            "enhanced": PipelineSpec(enhanced_config(), preset="enhanced")}


def expand_preset(name: str) -> PipelineSpec:
    presets = preset_specs()
    if name not in presets:
        raise ValidationError(f"unknown preset {name!r} (have: {', '.join(sorted(presets))})")
    return presets[name]


# ---------------------------------------------------------------------------
# device core
# ---------------------------------------------------------------------------

def _kernel_ready(pair: engine.DevicePair, gauss: bool) -> engine.DevicePair:
    """Float64 block means feed the fp32 Gaussian kernel as float32 (re-laid out aligned)."""
    if gauss and pair.code == nat.F64:
        return engine.device_pair(pair.ref.float(), pair.dist.float(), pair.bit_depth, True)
    return pair


def luma_records(pair: engine.DevicePair, config: SsimConfig, factor: Optional[int] = None,
                 stream=None, strict: bool = True) -> FrameRecords:
    """Luma-model records of a device batch (src/pipeline.py:213-236) without leaving the GPU.

    ``factor`` overrides the config's scale policy (None: derive it from the frame size).
    """
    n, h, w = pair.shape
    if factor is None:
        factor = policy_factor(config.scaling, w, h)
    win = config.window
    pair = _kernel_ready(downsample_pair(pair, factor, stream), win.shape == "gauss")
    _, h, w = pair.shape
    check_fit(h, w, win.k)
    resolve_engine(win, config.engine)
    spec = config.multiscale
    if spec.enabled:
        if min(h, w) // (1 << (spec.levels - 1)) < win.k:
            raise TooManyLevels(f"a {win.k}x{win.k} window does not fit the coarsest of {spec.levels} scales "
                                f"of a {w}x{h} image")
        _, score, _ = engine.msssim_levels(pair, win, config.c1, config.c2, spec.levels, spec=spec, stream=stream)
        return FrameRecords(score)
    pool = parse_spatial(config.spatial_pool)
    gh, gw = engine.grid_shape(h, w, win.k, win.stride)
    want = nat.WANT_Q | nat.WANT_L | nat.WANT_CS
    if pool.kind == "am":
        sums, _ = engine.ssim(pair, win, config.c1, config.c2, want, stream)
        means = engine.frame_means(sums, gh * gw)
        return FrameRecords(means[:, 0], means[:, 0], means[:, 1], means[:, 2])
    if win.shape == "rect" and (pool.kind == "cov" or (pool.kind == "md" and pool.p == 2.0)):
        # dispersion of the map from sum q and sum q^2 accumulated inside the rect kernel
        # (exact integer moments there; no map is written, no pooling pass): the
        # one-pass variance differs from numpy's two-pass std by ~1e-11 relative
        torch = nat.torch_mod()
        sums, _ = engine.ssim(pair, win, config.c1, config.c2, want | nat.WANT_Q2, stream)
        pooled = torch.empty((n,), dtype=torch.float64, device=sums.device)
        means = torch.empty((n, 3), dtype=torch.float64, device=sums.device)
        native = pool.native()
        rc = nat.lib().ssk_pool_moments(sums.data_ptr(), n, float(gh * gw), ctypes.byref(native), pooled.data_ptr(),
                                        means.data_ptr(), nat.stream_handle(stream))
        nat.raise_for(rc, "moment pooling")
        if strict and pool.kind == "cov" and bool(torch.isnan(pooled).any()):
            from .errors import ZeroMeanCoV

            raise ZeroMeanCoV("coefficient of variation is undefined for a zero-mean input")
        return FrameRecords(pooled, means[:, 0], means[:, 1], means[:, 2])
    sums, maps = engine.ssim(pair, win, config.c1, config.c2, want | nat.MAP_TERMS, stream)
    mu1 = None
    if pool.kind == "lw":
        _, stats = engine.ssim(pair, win, config.c1, config.c2, nat.MAP_STATS, stream)
        mu1 = stats[:, 0]
    pooled, _ = pool_maps(maps[:, 2], pool, mu1, stream=stream, strict=strict)
    means = engine.frame_means(sums, gh * gw)
    return FrameRecords(pooled, means[:, 0], means[:, 1], means[:, 2])


def score_batch(ref, dist, config: SsimConfig = SsimConfig(), stream=None) -> FrameRecords:
    """Batched luma pipeline on [n, h, w] CUDA tensors: scaling + SSIM/MS-SSIM + spatial pooling.

    Asynchronous (no host synchronisation); a zero-mean map under ``cov``
    pooling yields NaN for that frame instead of raising ZeroMeanCoV.
    """
    if config.color.model != "luma":
        raise ValidationError("score_batch scores luma planes; use color_batch for the channel-wise models")
    pair = engine.device_pair(ref, dist, config.bit_depth, config.window.shape == "gauss")
    return luma_records(pair, config, stream=stream, strict=False)


# ---------------------------------------------------------------------------
# single pair (reference signature)
# ---------------------------------------------------------------------------

def _luma_plane(frame):
    """``_luma_plane`` (src/pipeline.py:164-169): Y of YCbCr, BT.709 luma of RGB."""
    from .chroma import luma_of
    from .planes import SPACE_YCBCR, ColorFrame, LumaPlane

    if not isinstance(frame, ColorFrame):
        return frame
    if frame.space == SPACE_YCBCR:
        return LumaPlane(frame.channels[0], frame.bit_depth)
    return luma_of(frame)


def score_frame_pair(ref, dist, config: SsimConfig, volume=None) -> FrameScore:
    """Score one frame pair under a config (src/pipeline.py:197-258) on the device.

    Luma model: resolution adaptation, SSIM with the configured spatial pooler
    or MS-SSIM (score only), or SSIM-3D when a ``RollingVolume`` is given.
    Color models ``cw`` / ``fixed`` (channel-wise) and ``qssim`` / ``cmssim`` /
    ``hssim`` (colorimetric, ``colorimetric.py``) on YCbCr/RGB frames.
    """
    from . import chroma
    from .planes import ColorFrame, plane_bit_depth, plane_data, validate_color_pair, validate_frame_pair

    color_ref, color_dist = isinstance(ref, ColorFrame), isinstance(dist, ColorFrame)
    if color_ref != color_dist:
        raise DimensionMismatch("one stream is luma-only, the other tri-channel")
    if color_ref:
        validate_color_pair(ref, dist)
    else:
        ref, dist = validate_frame_pair(ref, dist)
    y1, y2 = _luma_plane(ref), _luma_plane(dist)
    yh, yw = plane_data(y1).shape
    factor = policy_factor(config.scaling, yw, yh)
    model = config.color.model
    if model == "luma":
        cfg = config.for_bit_depth(plane_bit_depth(y1, config.bit_depth))
        if volume is not None:
            if cfg.multiscale.enabled:
                raise ValidationError("use run_score for multiscale 3-D pipelines")
            return _volume_score(volume, scale_frame(y1, factor), scale_frame(y2, factor), cfg)
        pair = engine.upload_pair(plane_data(y1), plane_data(y2), cfg.bit_depth, cfg.window.shape == "gauss")
        return luma_records(pair, cfg, factor).host(0)
    if not color_ref:
        raise ValidationError(f"color model {model!r} needs tri-channel input, stream is luma-only")
    ref, dist = scale_frame(ref, factor), scale_frame(dist, factor)
    cfg = config.for_bit_depth(ref.bit_depth)
    if model == "cw":
        return FrameScore(chroma.channelwise_cssim(ref, dist, cfg.color.alpha, cfg.color.beta, cfg), None, None, None)
    if model == "fixed":
        return FrameScore(chroma.fixed_weight_cssim(ref, dist, cfg.color.weights, cfg), None, None, None)
    from . import colorimetric as cm

    if model == "qssim":
        pair = (ref, dist)
        if cfg.color.space in ("rgb", "lab") and ref.space != "rgb":
            pair = (cm.ycbcr_bt709_to_rgb(ref), cm.ycbcr_bt709_to_rgb(dist))
        score = cm.qssim(*pair, window=cfg.window, k1=cfg.k1, k2=cfg.k2, space=cfg.color.space)
    elif model == "cmssim":
        score = cm.cmssim(ref, dist, cfg.window, cfg)
    else:  # hssim
        score = cm.hssim(ref, dist, cfg.window, cfg)
    return FrameScore(score, None, None, None)


def _volume_score(volume, y1, y2, cfg: SsimConfig) -> FrameScore:
    """SSIM-3D record for one pushed frame (src/pipeline.py:217-223, :229-236)."""
    volume.push(y1, y2)
    pool = parse_spatial(cfg.spatial_pool)
    if pool.kind == "am":
        q, lm, cm = volume.terms(cfg.window, cfg)
        return FrameScore(q, q, lm, cm)
    maps = volume._run(cfg.window, cfg.c1, cfg.c2, nat.WANT_Q | nat.WANT_L | nat.WANT_CS | nat.MAP_TERMS)
    sums, terms, (gh, gw) = maps
    means = engine.frame_means(sums, gh * gw)[0].cpu().numpy()
    mu1 = None
    if pool.kind == "lw":
        _, stats, _ = volume._run(cfg.window, 1.0, 1.0, nat.MAP_STATS)
        mu1 = stats[:, 0]
    pooled, _ = pool_maps(terms[:, 2], pool, mu1)
    return FrameScore(float(pooled[0].item()), float(means[0]), float(means[1]), float(means[2]))


# ---------------------------------------------------------------------------
# whole-run driver (src/pipeline.py:261-366)
# ---------------------------------------------------------------------------

def _user_seconds() -> tuple[float, str]:
    try:
        import resource

        return resource.getrusage(resource.RUSAGE_SELF).ru_utime, "user"
    except ImportError:  # no resource module: wall time
        import time

        return time.perf_counter(), "wall"


def run_score(ref_path, dist_path, spec: PipelineSpec, *, width: Optional[int] = None, height: Optional[int] = None,
              bit_depth: int = 8, chroma: str = "420", batch_frames: int = 16) -> dict:
    """Score two media files: {"records": per-frame dicts (FRAME_FIELDS), "summary": {...}}.

    Luma pipelines over Y4M / raw streams run batched: memory-mapped planes ->
    pinned double buffer -> device (``SequenceScorer``), ``batch_frames`` frames
    per launch; SSIM-3D (kt > 1), the color models and still images go frame by
    frame through ``score_frame_pair`` (all on the device).
    """
    import time

    import numpy as np

    from .errors import DimensionMismatch, LengthMismatch, SsimkitError
    from .ingest import VideoStream, open_stream
    from .planes import ScoreSeries
    from .pooling import pool_temporal
    from .volume import RollingVolume, msssim3d

    ref = open_stream(ref_path, width, height, bit_depth, chroma)
    dist = open_stream(dist_path, width, height, bit_depth, chroma)
    if isinstance(ref, VideoStream) and isinstance(dist, VideoStream):
        rh, dh = ref.header, dist.header
        if (rh.width, rh.height) != (dh.width, dh.height):
            raise DimensionMismatch(f"{ref_path} is {rh.width}x{rh.height}, {dist_path} is {dh.width}x{dh.height}")
        if rh.bit_depth != dh.bit_depth or rh.chroma != dh.chroma:
            raise DimensionMismatch("streams differ in bit depth or chroma subsampling")
        if len(ref) != len(dist):
            raise LengthMismatch(f"streams differ in length ({len(ref)} vs {len(dist)} frames)")
    elif len(ref) != len(dist):
        raise LengthMismatch("streams differ in length")
    config = spec.config
    start, timing_source = _user_seconds()
    wall0 = time.perf_counter()
    results: list = []
    try:
        batched = (spec.kt == 1 and config.color.model == "luma" and isinstance(ref, VideoStream)
                   and isinstance(dist, VideoStream))
        if batched:
            from .video import SequenceScorer

            cfg = config.for_bit_depth(ref.header.bit_depth)
            from .ingest import pinned_pair

            with pinned_pair(ref.source, dist.source) as direct:  # DMA straight from page-locked mappings
                seq = SequenceScorer(cfg, batch_frames).score(ref.source.luma(), dist.source.luma(),
                                                              direct=direct)
            results = [FrameScore(r.score, r.am, r.l_mean, r.cs_mean) for r in seq.records]
        elif spec.kt > 1 and config.multiscale.enabled:
            series = msssim3d(_luma_iter(ref), _luma_iter(dist), spec.kt, config.multiscale, config)
            results = [FrameScore(float(x), None, None, None) for x in series.scores]
        else:
            volume = RollingVolume(spec.kt) if spec.kt > 1 else None
            for i, (a, b) in enumerate(zip(ref, dist)):
                try:
                    results.append(score_frame_pair(a, b, config, volume))
                except SsimkitError as exc:
                    raise type(exc)(f"frame {i}: {exc}") from exc
    except SsimkitError as exc:
        raise type(exc)(f"{ref_path} vs {dist_path}: {exc}") from exc
    if not results:
        raise ValidationError(f"{ref_path} vs {dist_path}: no frames to score")
    end, _ = _user_seconds()
    elapsed = end - start if timing_source == "user" else time.perf_counter() - wall0
    records = [{"frame": i, "score": r.score, "am": r.am, "l_mean": r.l_mean, "cs_mean": r.cs_mean}
               for i, r in enumerate(results)]
    scores = np.array([r.score for r in results], dtype=np.float64)
    summary = {"frames": len(results), "spatial_pool": config.spatial_pool, "temporal_pool": config.temporal_pool,
               "pooled_score": pool_temporal(ScoreSeries(scores), config.temporal_pool),
               "mean_score": float(scores.mean()), "user_seconds": elapsed, "timing_source": timing_source}
    ams = [r.am for r in results if r.am is not None]
    if ams:
        summary["mean_am"] = float(np.mean(ams))
    if parse_spatial(config.spatial_pool).kind == "cov":
        summary["note"] = ("cov pooling maps a perfect (constant 1) quality map to 0; "
                           "per-frame arithmetic means are reported in the 'am' field")
    return {"records": records, "summary": summary}


def _luma_iter(stream):
    from .ingest import VideoStream

    if isinstance(stream, VideoStream):
        return stream.luma_frames()
    return (_luma_plane(f) for f in stream)
