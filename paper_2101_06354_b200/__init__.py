"""B200-native SSIM engine: a drop-in for ssimkit's SSIM / MS-SSIM hot path.

Reference: ssimkit (arXiv 2101.06354, "A Hitchhiker's Guide to Structural
Similarity"), /root/reference/pkg/src/ssimkit.  The names below keep the
reference's public API for the accelerated path (its ``__all__``,
src/__init__.py:68-135): window statistics, SSIM maps and scores, MS-SSIM,
channel-wise color SSIM, pooling, and the configuration/container types.
All computation runs in hand-written sm_100a CUDA kernels (libssimk.so,
C ABI in include/ssimk.h); there is no CPU fallback.

New API for throughput: ``ssim_batch`` / ``msssim_batch`` / ``color_batch``
on [n, h, w] CUDA tensors, and ``SequenceScorer`` for frame streams.
"""

from .batch import FrameTerms, HostBatchScorer, color_batch, msssim_batch, ssim_batch, ssim_terms_batch
from .chroma import (
    channel_scores,
    channelwise_cssim,
    combine_channelwise,
    fixed_weight_cssim,
    luma_of,
    rgb_to_ycbcr_bt709,
    upsample_chroma,
    ycbcr_bt709_to_rgb,
)
from .colorimetric import cmssim, delta_e_map, hssim, hue_plane, qssim
from .errors import SsimkitError
from .moments import (
    IntegralSet,
    LocalStatsMaps,
    build_integral_set,
    gaussian_kernel,
    local_statistics,
    rect_equivalent,
    stats_from_sums,
    window_sum,
)
from .options import (
    STANDARD_EXPONENTS,
    ColorModelSpec,
    MultiscaleSpec,
    ScalePolicy,
    SsimConfig,
    WindowSpec,
    parse_color,
    parse_multiscale,
    parse_scale,
    parse_window,
)
from .planes import ColorFrame, LumaPlane, QualityMap, ScoreSeries, validate_frame_pair
from .pooling import SpatialPooler, TemporalPooler, parse_spatial, parse_temporal, pool_maps, pool_spatial, pool_temporal
from .adaptation import (
    box_downsample,
    enhanced_scale_factor,
    legacy_scale_factor,
    policy_factor,
    round_half_away,
    sast_factor,
    viewing_geometry,
)
from .pipeline import (
    FRAME_FIELDS,
    FrameRecords,
    PipelineSpec,
    expand_preset,
    luma_records,
    preset_specs,
    run_score,
    score_batch,
)
from .pyramid import combine_scale_scores, dyadic_downsample, msssim, scale_scores
from .scoring import (
    SsimTermMaps,
    mssim,
    ssim_map,
    ssim_score,
    ssim_terms,
    term_maps_from_stats,
    weber_contrast_term,
    weber_luminance_term,
)
from .video import FrameScore, SequenceScorer, gather_frame_scores, score_frame_pair, score_sequence, shard_bounds
from .ingest import (
    FrameSource,
    StreamHeader,
    VideoStream,
    format_float,
    open_raw,
    open_stream,
    open_y4m,
    read_planar_raw,
    read_pnm,
    read_y4m,
    score_files,
    write_planar_raw,
    write_report,
    write_y4m,
)
from .volume import (
    REFRESH_INTERVAL,
    RollingVolume,
    msssim3d,
    push_frame,
    shard_with_halo,
    ssim3d_map,
    ssim3d_series,
    ssim3d_series_shard,
)

__version__ = "0.1.0"

__all__ = [
    # configuration
    "ColorModelSpec", "MultiscaleSpec", "ScalePolicy", "SsimConfig", "STANDARD_EXPONENTS", "WindowSpec",
    "parse_color", "parse_multiscale", "parse_scale", "parse_window",
    # containers / errors
    "ColorFrame", "LumaPlane", "QualityMap", "ScoreSeries", "validate_frame_pair", "SsimkitError",
    # local statistics
    "IntegralSet", "LocalStatsMaps", "build_integral_set", "gaussian_kernel", "local_statistics",
    "rect_equivalent", "stats_from_sums", "window_sum",
    # SSIM
    "SsimTermMaps", "mssim", "ssim_map", "ssim_score", "ssim_terms", "term_maps_from_stats",
    "weber_luminance_term", "weber_contrast_term",
    # multiscale
    "combine_scale_scores", "dyadic_downsample", "msssim", "scale_scores",
    # color
    "channel_scores", "channelwise_cssim", "combine_channelwise", "fixed_weight_cssim", "luma_of",
    "rgb_to_ycbcr_bt709", "upsample_chroma", "ycbcr_bt709_to_rgb",
    "cmssim", "delta_e_map", "hssim", "hue_plane", "qssim",
    # pooling
    "SpatialPooler", "TemporalPooler", "parse_spatial", "parse_temporal", "pool_maps", "pool_spatial",
    "pool_temporal",
    # resolution adaptation
    "box_downsample", "enhanced_scale_factor", "legacy_scale_factor", "policy_factor", "round_half_away",
    "sast_factor", "viewing_geometry",
    # pipeline contract / presets
    "FRAME_FIELDS", "FrameRecords", "PipelineSpec", "expand_preset", "luma_records", "preset_specs", "run_score",
    "score_batch",
    # batched device API / sequences / multi-GPU
    "FrameTerms", "HostBatchScorer", "color_batch", "msssim_batch", "ssim_batch", "ssim_terms_batch",
    "SequenceScorer", "gather_frame_scores", "score_sequence", "shard_bounds", "FrameScore", "score_frame_pair",
    # media ingest
    "FrameSource", "StreamHeader", "VideoStream", "format_float", "open_raw", "open_stream", "open_y4m",
    "read_planar_raw", "read_pnm", "read_y4m", "score_files", "write_planar_raw", "write_report", "write_y4m",
    # spatio-temporal (SSIM-3D)
    "REFRESH_INTERVAL", "RollingVolume", "msssim3d", "push_frame", "ssim3d_map", "ssim3d_series",
    "shard_with_halo", "ssim3d_series_shard",
]
