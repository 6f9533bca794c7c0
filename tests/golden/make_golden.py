"""Generate golden vectors by running the REFERENCE (ssimkit) itself.

Run in the build container, where the read-only reference is importable:

    PYTHONPATH=/root/reference/pkg/src python -B tests/golden/make_golden.py

Writes tests/golden/golden_v1.npz (inputs + the reference's outputs for
small seeded cases covering every hot-path entry point: Gaussian / rect /
strided / 10-bit / 16-bit / float windows, exact int64 window sums and
summed-area tables, the dyadic pyramid, MS-SSIM product/sum/fast4, the
channel-wise color models on 4:2:0 frames, temporal mean pooling and the
config-1 512x512 score).  The GPU box has no /root/reference: tests there
read these fixtures and the oracle (pinned against them) instead.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

import ssimkit  # noqa: E402  (the reference, from PYTHONPATH)
from ssimkit.config import MultiscaleSpec, SsimConfig, WindowSpec  # noqa: E402
from ssimkit.frames import ColorFrame, LumaPlane  # noqa: E402
from ssimkit.multiscale import dyadic_downsample, msssim, scale_scores  # noqa: E402
from ssimkit.stats import TABLE_IDS, _grid_window_sums, build_integral_set, local_statistics  # noqa: E402
from ssimkit.ssim import mssim, ssim_map  # noqa: E402
from ssimkit.color import channelwise_cssim, fixed_weight_cssim  # noqa: E402
from ssimkit.pooling import pool_temporal  # noqa: E402

from paper_2101_06354_b200 import synth  # noqa: E402  (seeded input generators, numpy only)


def natural(rng, h, w, peak=255.0, dtype=np.uint8):
    return synth.inv_f_noise(rng, h, w, peak).astype(dtype)


def noisy(rng, a, amp, peak):
    return np.clip(a.astype(np.int64) + rng.integers(-amp, amp + 1, a.shape), 0, peak).astype(a.dtype)


def main() -> None:
    rng = np.random.default_rng(20240117)
    out: dict[str, np.ndarray] = {}

    def put_maps(name, a, b, cfg, bd=8):
        ra, rb = LumaPlane(a, bd), LumaPlane(b, bd)
        maps = ssim_map(ra, rb, cfg)
        st = local_statistics(ra, rb, cfg.window, cfg.engine)
        out[f"{name}/ref"] = a
        out[f"{name}/dist"] = b
        out[f"{name}/l"] = maps.l_map.values
        out[f"{name}/cs"] = maps.cs_map.values
        out[f"{name}/q"] = maps.q_map.values
        out[f"{name}/stats"] = np.stack([st.mu1, st.mu2, st.var1, st.var2, st.cov])
        out[f"{name}/score"] = np.array(mssim(maps))
        out[f"{name}/terms"] = np.array([maps.q_map.values.mean(), maps.l_map.values.mean(),
                                         maps.cs_map.values.mean()])

    # Gaussian 11 / 1.5 (the canonical window), 8-bit
    a = natural(rng, 48, 64)
    put_maps("gauss11", a, noisy(rng, a, 20, 255), SsimConfig(window=WindowSpec.gaussian(1.5)))
    # Gaussian strided
    a = natural(rng, 41, 53)
    put_maps("gauss_s3", a, noisy(rng, a, 25, 255), SsimConfig(window=WindowSpec.gaussian(1.5, stride=3)))
    # Gaussian sigma 2 (k = 13), 10-bit
    a = natural(rng, 40, 44, 1023.0, np.uint16)
    put_maps("gauss13_10b", a, noisy(rng, a, 60, 1023), SsimConfig(bit_depth=10, window=WindowSpec.gaussian(2.0)), bd=10)
    # default config: rect 11, integral engine
    a = natural(rng, 37, 45)
    put_maps("rect11", a, noisy(rng, a, 30, 255), SsimConfig())
    # rect 8 stride 4, 10-bit (config-4 shape, small)
    a = natural(rng, 64, 80, 1023.0, np.uint16)
    b = noisy(rng, a, 40, 1023)
    put_maps("rect8s4_10b", a, b, SsimConfig(bit_depth=10, window=WindowSpec.rectangular(8, stride=4), engine="integral"), bd=10)
    iset = build_integral_set(LumaPlane(a, 10), LumaPlane(b, 10))
    out["rect8s4_10b/wsums"] = np.stack([_grid_window_sums(iset.table(t), 8, 4) for t in TABLE_IDS])
    # 16-bit full range, rect 11 (64-bit sums)
    a = rng.integers(0, 65536, (30, 40)).astype(np.uint16)
    b = rng.integers(0, 65536, (30, 40)).astype(np.uint16)
    put_maps("rect11_16b", a, b, SsimConfig(bit_depth=16), bd=16)
    iset = build_integral_set(LumaPlane(a, 16), LumaPlane(b, 16))
    out["rect11_16b/wsums"] = np.stack([_grid_window_sums(iset.table(t), 11, 1) for t in TABLE_IDS])
    # rect 1 and rect 16, naive engine
    a = natural(rng, 24, 30)
    put_maps("rect1", a, noisy(rng, a, 9, 255), SsimConfig(window=WindowSpec.rectangular(1), engine="naive"))
    a = natural(rng, 33, 35)
    put_maps("rect16", a, noisy(rng, a, 9, 255), SsimConfig(window=WindowSpec.rectangular(16), engine="naive"))
    # float planes (5-point blurred), rect 5
    a = natural(rng, 26, 31).astype(np.float64)
    b = (np.roll(a, 1, 0) + np.roll(a, -1, 0) + np.roll(a, 1, 1) + np.roll(a, -1, 1) + a) / 5.0
    put_maps("rect5_float", a, b, SsimConfig(window=WindowSpec.rectangular(5)))

    # summed-area tables (7 x 5) and a 2x2 downsample
    a = rng.integers(0, 256, (7, 5)).astype(np.uint8)
    b = rng.integers(0, 256, (7, 5)).astype(np.uint8)
    iset = build_integral_set(LumaPlane(a), LumaPlane(b))
    out["sat/ref"], out["sat/dist"] = a, b
    out["sat/tables"] = np.stack([iset.table(t) for t in TABLE_IDS])
    a = rng.integers(0, 256, (21, 34)).astype(np.uint8)
    out["down/in"] = a
    out["down/out"] = dyadic_downsample(LumaPlane(a)).samples

    # MS-SSIM: Gaussian 5 levels product, rect 5 (3 levels sum / fast4)
    a = natural(rng, 176, 208)
    b = noisy(rng, a, 25, 255)
    cfg = SsimConfig(window=WindowSpec.gaussian(1.5))
    out["ms_gauss/ref"], out["ms_gauss/dist"] = a, b
    out["ms_gauss/levels"] = np.array(scale_scores(LumaPlane(a), LumaPlane(b), cfg, 5))
    out["ms_gauss/score"] = np.array(msssim(LumaPlane(a), LumaPlane(b), cfg, MultiscaleSpec.product(5)))
    a = natural(rng, 96, 100)
    b = noisy(rng, a, 18, 255)
    cfg = SsimConfig(window=WindowSpec.rectangular(5))
    out["ms_rect5/ref"], out["ms_rect5/dist"] = a, b
    out["ms_rect5/levels4"] = np.array(scale_scores(LumaPlane(a), LumaPlane(b), cfg, 4))
    out["ms_rect5/sum3"] = np.array(msssim(LumaPlane(a), LumaPlane(b), cfg, MultiscaleSpec("sum", 3, (0.2, 0.3, 0.5))))
    out["ms_rect5/fast4"] = np.array(msssim(LumaPlane(a), LumaPlane(b), cfg, MultiscaleSpec.fast4()))

    # color 4:2:0, channel-wise models
    y = natural(rng, 40, 48)
    c1 = natural(rng, 20, 24)
    c2 = natural(rng, 20, 24)
    ref = ColorFrame((y, c1, c2), "ycbcr-bt709", "420")
    dist = ColorFrame((noisy(rng, y, 12, 255), noisy(rng, c1, 20, 255), noisy(rng, c2, 6, 255)), "ycbcr-bt709", "420")
    cfg = SsimConfig(window=WindowSpec.gaussian(1.5))
    for i, (r, d) in enumerate(zip(ref.channels, dist.channels)):
        out[f"color/ref{i}"], out[f"color/dist{i}"] = r, d
    out["color/fixed"] = np.array(fixed_weight_cssim(ref, dist, (4 / 6, 1 / 6, 1 / 6), cfg))
    out["color/cw"] = np.array(channelwise_cssim(ref, dist, -0.3, -0.3, cfg))
    out["color/per_plane"] = np.array([mssim(ssim_map(r, d, cfg)) for r, d in zip(ref.channels, dist.channels)])

    # temporal am pooling of a score series
    series = rng.uniform(0.5, 1.0, 37)
    out["temporal/series"] = series
    out["temporal/am"] = np.array(pool_temporal(series, "am"))

    # config 1 (512 x 512 u8, Gaussian 11/1.5): score only; inputs regenerated from the seed
    a, b = synth.config1_pair()
    maps = ssim_map(LumaPlane(a), LumaPlane(b), SsimConfig(window=WindowSpec.gaussian(1.5)))
    out["config1/sha256"] = np.frombuffer(hashlib.sha256(a.tobytes() + b.tobytes()).digest(), dtype=np.uint8)
    out["config1/terms"] = np.array([maps.q_map.values.mean(), maps.l_map.values.mean(), maps.cs_map.values.mean()])

    # SSIM-3D rolling volumes (src/spatiotemporal.py): integer and float streams,
    # a refresh inside the float run, and the multiscale variant
    from ssimkit.spatiotemporal import RollingVolume, msssim3d, ssim3d_map, ssim3d_series

    frames_a = [natural(rng, 36, 44) for _ in range(7)]
    frames_b = [noisy(rng, f, 15, 255) for f in frames_a]
    for i in range(7):
        out[f"vol/ref{i}"], out[f"vol/dist{i}"] = frames_a[i], frames_b[i]
    out["vol/series_k3"] = ssim3d_series([LumaPlane(f) for f in frames_a], [LumaPlane(f) for f in frames_b], 3,
                                         SsimConfig(window=WindowSpec.rectangular(7))).scores
    out["vol/series_k1"] = ssim3d_series([LumaPlane(f) for f in frames_a], [LumaPlane(f) for f in frames_b], 1,
                                         SsimConfig(window=WindowSpec.rectangular(5, stride=2))).scores
    vol = RollingVolume(4)
    for fa, fb in zip(frames_a, frames_b):
        vol.push(LumaPlane(fa), LumaPlane(fb))
    st = vol.local_statistics(WindowSpec.rectangular(6))
    out["vol/stats_k4_w6"] = np.stack([st.mu1, st.mu2, st.var1, st.var2, st.cov])
    maps = ssim3d_map(vol, WindowSpec.rectangular(6), SsimConfig())
    out["vol/q_k4_w6"] = maps.q_map.values
    fl_a = [f.astype(np.float64) / 3.0 for f in frames_a]
    fl_b = [f.astype(np.float64) / 3.0 for f in frames_b]
    volf = RollingVolume(3, refresh_interval=4)
    series = []
    for fa, fb in zip(fl_a, fl_b):
        volf.push(fa, fb)
        series.append(float(ssim3d_map(volf, WindowSpec.rectangular(5)).q_map.values.mean()))
    out["vol/series_float_refresh4"] = np.array(series)
    big_a = [natural(rng, 48, 52) for _ in range(4)]
    big_b = [noisy(rng, f, 20, 255) for f in big_a]
    for i in range(4):
        out[f"vol/msref{i}"], out[f"vol/msdist{i}"] = big_a[i], big_b[i]
    out["vol/ms3d"] = msssim3d([LumaPlane(f) for f in big_a], [LumaPlane(f) for f in big_b], 2,
                               MultiscaleSpec.product(3), SsimConfig(window=WindowSpec.rectangular(5))).scores

    np.savez_compressed(HERE / "golden_v1.npz", **out)
    print(f"wrote {len(out)} arrays, reference ssimkit {ssimkit.__version__}")


if __name__ == "__main__":
    main()
