"""Golden vectors for spatial pooling, resolution adaptation and the per-frame
pipeline record, produced by running the REFERENCE (ssimkit) itself.

    PYTHONPATH=/root/reference/pkg/src python -B tests/golden/make_golden_pool.py

Writes tests/golden/golden_pool_v1.npz:
  pool/<map>/values (+ /luma)          quality maps (seeded, with ties and edge cases)
  pool/<map>/<selector>                 pool_spatial(values, selector[, ref_luma]) (src/pooling.py:202)
  down/<case>/in, down/<case>/f<k>      box_downsample(plane, k) (src/adaptation.py:93)
  factor/table                          policy_factor for sizes x policies (src/adaptation.py:81)
  frame/<case>/record                   score_frame_pair(...) = (score, am, l_mean, cs_mean)
                                        (src/pipeline.py:197), inputs regenerated from the seeds
                                        in frame/<case>/seed with paper_2101_06354_b200.synth
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

from ssimkit.adaptation import box_downsample, policy_factor  # noqa: E402  (the reference)
from ssimkit.config import ScalePolicy, SsimConfig, WindowSpec  # noqa: E402
from ssimkit.frames import LumaPlane  # noqa: E402
from ssimkit.pipeline import expand_preset, score_frame_pair  # noqa: E402
from ssimkit.pooling import pool_spatial  # noqa: E402

from paper_2101_06354_b200 import synth  # noqa: E402

SELECTORS = ("am", "cov", "md", "md:p=3,o=2", "md:p=1,o=0.5", "fns", "dw", "dw:p=2.5", "mink", "mink:p=3",
             "pp", "pp:ps=6,rs=4", "pp:ps=37.5,rs=1000", "pp:ps=100,rs=2", "pp:ps=0,rs=5",
             "lw:a=10,b=5", "lw:a=60,b=0")

DOWN_FACTORS = (1, 2, 3, 4, 5, 6, 7, 9, 12, 17)

# sizes (w, h) x policies for the factor table
SIZES = ((176, 144), (352, 288), (640, 480), (720, 576), (1280, 720), (1920, 1080), (2560, 1440),
         (3840, 2160), (300, 200), (383, 1000))
POLICIES = (ScalePolicy.none(), ScalePolicy.legacy256(), ScalePolicy.legacy256("ceil"), ScalePolicy.enhanced_dh(3.0),
            ScalePolicy.enhanced_dh(1.5), ScalePolicy.enhanced_dh(6.0), ScalePolicy.sast(1000.0),
            ScalePolicy.sast(2500.0, 30.0, 45.0))

# per-frame pipeline cases: (name, h, w, bit depth, config, seed)
FRAME_CASES = (
    ("enh_1080", 1080, 1920, 8, "enhanced", 7001),
    ("enh_720", 720, 1280, 8, "enhanced", 7002),
    ("enh_576_10b", 576, 720, 10, "enhanced", 7003),
    ("legacy_gauss_fns", 600, 800, 8, ("legacy", "gauss", "fns"), 7004),
    ("rect_pp", 96, 128, 8, ("none", "rect", "pp:ps=10,rs=4"), 7005),
    ("gauss_md", 90, 120, 8, ("none", "gauss", "md:p=2,o=1"), 7006),
    ("rect_lw", 80, 100, 8, ("none", "rect", "lw:a=40,b=20"), 7007),
    ("gauss_dw", 72, 88, 8, ("none", "gauss", "dw:p=2"), 7008),
)


def frame_inputs(h: int, w: int, bd: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """Seeded natural-image pair (1/f noise + bounded noise), regenerated the same way by the tests."""
    rng = np.random.default_rng(seed)
    peak = float((1 << bd) - 1)
    dt = np.uint8 if bd == 8 else np.uint16
    a = synth.inv_f_noise(rng, h, w, peak).astype(dt)
    amp = 12 * (1 << (bd - 8))
    b = np.clip(a.astype(np.int64) + rng.integers(-amp, amp + 1, a.shape), 0, int(peak)).astype(dt)
    return a, b


def big_map() -> tuple[np.ndarray, np.ndarray]:
    """700 x 900 heavy-tailed quality map + luma map from seed 4343 (same recipe in the tests)."""
    rng = np.random.default_rng(4343)
    v = np.clip(1.0 - np.abs(rng.standard_cauchy((700, 900))) * 0.01, -1.0, 1.0)
    return v, rng.uniform(0.0, 120.0, v.shape)


def frame_config(spec, bd: int) -> SsimConfig:
    if spec == "enhanced":
        return expand_preset("enhanced").config.for_bit_depth(bd)
    scaling, window, pool = spec
    win = WindowSpec.gaussian(1.5) if window == "gauss" else WindowSpec.rectangular(11)
    pol = ScalePolicy.legacy256() if scaling == "legacy" else ScalePolicy.none()
    return SsimConfig(bit_depth=bd, window=win, scaling=pol, spatial_pool=pool)


def main() -> None:
    rng = np.random.default_rng(4242)
    out: dict[str, np.ndarray] = {}

    maps = {
        "ssimlike": np.clip(1.0 - np.abs(rng.normal(0.0, 0.08, (53, 71))), -1.0, 1.0),
        "ties": np.round(rng.uniform(-0.2, 1.0, (40, 37)), 2),          # many duplicated values
        "wide": rng.uniform(-0.5, 1.0, (3, 1500)),
        "tall": rng.uniform(0.0, 1.0, (1200, 2)),
        "ones": np.ones((9, 11)),                                       # dw's all-ones fallback
        "single": np.array([[0.37]]),
        "pair": np.array([[0.9, -0.1]]),
    }
    for name, v in maps.items():
        luma = rng.uniform(0.0, 120.0, v.shape)
        out[f"pool/{name}/values"] = v
        out[f"pool/{name}/luma"] = luma
        for sel in SELECTORS:
            out[f"pool/{name}/{sel}"] = np.array(pool_spatial(v, sel, ref_luma=luma))
    # a large map (not stored: regenerated from its seed by big_map())
    v, luma = big_map()
    for sel in SELECTORS:
        out[f"pool/big/{sel}"] = np.array(pool_spatial(v, sel, ref_luma=luma))

    planes = {
        "u8": rng.integers(0, 256, (37, 53)).astype(np.uint8),
        "u16": rng.integers(0, 1024, (64, 45)).astype(np.uint16),
        "even": rng.integers(0, 256, (48, 64)).astype(np.uint8),
        "f64": rng.uniform(0.0, 255.0, (29, 31)),
        "f64big": rng.uniform(0.0, 1023.0, (61, 75)),
    }
    for name, a in planes.items():
        out[f"down/{name}/in"] = a
        for f in DOWN_FACTORS:
            out[f"down/{name}/f{f}"] = np.asarray(box_downsample(a, f), dtype=np.float64)

    table = np.array([[policy_factor(pol, w, h) for pol in POLICIES] for (w, h) in SIZES], dtype=np.int64)
    out["factor/table"] = table

    for name, h, w, bd, spec, seed in FRAME_CASES:
        a, b = frame_inputs(h, w, bd, seed)
        cfg = frame_config(spec, bd)
        rec = score_frame_pair(LumaPlane(a, bd), LumaPlane(b, bd), cfg)
        vals = [rec.score, rec.am, rec.l_mean, rec.cs_mean]
        out[f"frame/{name}/record"] = np.array([np.nan if x is None else x for x in vals], dtype=np.float64)
        out[f"frame/{name}/seed"] = np.array([seed, h, w, bd])
        print(name, vals)

    np.savez_compressed(HERE / "golden_pool_v1.npz", **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
