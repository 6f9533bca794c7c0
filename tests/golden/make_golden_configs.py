"""Full-size golden SCORES for the BASELINE.json configurations, made by running the REFERENCE.

Run in the build container, where the read-only reference is importable:

    PYTHONPATH=/root/reference/pkg/src python -B tests/golden/make_golden_configs.py [--workers 8]

Only scalars are stored (the frames are regenerated from ``synth``'s seeds on the
GPU box, and each frame's CRC32 is stored next to its scores so a test can tell
"the synthetic input changed" apart from "the engine is wrong"):

* config 2 -- all 64 pairs of 1080p u8: Gaussian 11/1.5 ``ssim_map`` means
  (score, l_mean, cs_mean), the 5 ``scale_scores`` and ``msssim`` (product, standard
  exponents); plus ``msssim`` under the reference's default window (rect 11, auto engine);
* config 3 -- all 300 YUV420 1080p frames: per-plane ``mssim(ssim_map(..))`` scores,
  ``fixed_weight_cssim`` with weights (4/6, 1/6, 1/6) and ``pool_temporal(.., "am")``;
* config 4 -- 4 pairs of 4K 10-bit: rect 8 stride 4 integral ``ssim_map`` means;
* config 5 -- 8 pairs of 4K u8: Gaussian SSIM terms, 5 scale scores and ``msssim``.

Writes tests/golden/golden_configs_v1.npz.
"""

from __future__ import annotations

import argparse
import sys
import time
import zlib
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

from paper_2101_06354_b200 import synth  # noqa: E402  (seeded input generators)

C3_WEIGHTS = (4 / 6, 1 / 6, 1 / 6)
C4_PAIRS = 4
C5_PAIRS = 8


def crc(*arrays) -> int:
    c = 0
    for a in arrays:
        c = zlib.crc32(np.ascontiguousarray(a).tobytes(), c)
    return c


def _gauss():
    from ssimkit.config import SsimConfig, WindowSpec

    return SsimConfig(window=WindowSpec.gaussian(1.5))


def _terms(a, b, cfg):
    from ssimkit.ssim import ssim_map

    m = ssim_map(a, b, cfg)
    return [float(m.q_map.values.mean()), float(m.l_map.values.mean()), float(m.cs_map.values.mean())]


def _dct_job(args):
    cfgno, i, h, w, with_rect = args
    from ssimkit.config import MultiscaleSpec, SsimConfig
    from ssimkit.multiscale import combine_scale_scores, msssim, scale_scores

    a, b = synth.dct_pair(cfgno, i, h, w)
    cfg = _gauss()
    spec = MultiscaleSpec.product(5)
    lv = scale_scores(a, b, cfg, 5)
    out = dict(crc=crc(a, b), terms=_terms(a, b, cfg), levels=lv, msssim=combine_scale_scores(lv, spec))
    if with_rect:
        out["msssim_rect11"] = msssim(a, b, SsimConfig(), spec)
    return out


_VID = None


def _vid_init():
    global _VID
    _VID = synth.VideoConfig3()


def _c3_job(t):
    from ssimkit.color import fixed_weight_cssim
    from ssimkit.frames import ColorFrame
    from ssimkit.ssim import mssim, ssim_map

    r, d = _VID.pair(t)
    cfg = _gauss()
    planes = [mssim(ssim_map(x, y, cfg)) for x, y in zip(r, d)]
    fixed = fixed_weight_cssim(ColorFrame(r, "ycbcr-bt709", "420"), ColorFrame(d, "ycbcr-bt709", "420"),
                               C3_WEIGHTS, cfg)
    return dict(crc=crc(*r, *d), planes=planes, score=fixed)


def _c4_job(i):
    from ssimkit.config import SsimConfig, WindowSpec
    from ssimkit.frames import LumaPlane

    a, b = synth.config4_pair(i)
    cfg = SsimConfig(bit_depth=10, window=WindowSpec.rectangular(8, stride=4), engine="integral")
    return dict(crc=crc(a, b), terms=_terms(LumaPlane(a, 10), LumaPlane(b, 10), cfg))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=8)
    args = ap.parse_args()
    out: dict[str, np.ndarray] = {}
    t0 = time.time()
    with ProcessPoolExecutor(args.workers) as ex:
        r2 = list(ex.map(_dct_job, [(2, i, 1080, 1920, True) for i in range(64)]))
        r5 = list(ex.map(_dct_job, [(5, i, 2160, 3840, False) for i in range(C5_PAIRS)]))
        r4 = list(ex.map(_c4_job, range(C4_PAIRS)))
    print(f"configs 2/4/5 done in {time.time() - t0:.0f} s", flush=True)
    with ProcessPoolExecutor(args.workers, initializer=_vid_init) as ex:
        r3 = list(ex.map(_c3_job, range(300), chunksize=4))
    print(f"config 3 done in {time.time() - t0:.0f} s", flush=True)
    from ssimkit.frames import ScoreSeries
    from ssimkit.pooling import pool_temporal

    for tag, rows in (("c2", r2), ("c5", r5)):
        out[f"{tag}/crc"] = np.array([r["crc"] for r in rows], np.uint32)
        out[f"{tag}/terms"] = np.array([r["terms"] for r in rows])
        out[f"{tag}/levels"] = np.array([r["levels"] for r in rows])
        out[f"{tag}/msssim"] = np.array([r["msssim"] for r in rows])
    out["c2/msssim_rect11"] = np.array([r["msssim_rect11"] for r in r2])
    out["c4/crc"] = np.array([r["crc"] for r in r4], np.uint32)
    out["c4/terms"] = np.array([r["terms"] for r in r4])
    out["c3/crc"] = np.array([r["crc"] for r in r3], np.uint32)
    out["c3/planes"] = np.array([r["planes"] for r in r3])
    out["c3/scores"] = np.array([r["score"] for r in r3])
    out["c3/pooled"] = np.array(pool_temporal(ScoreSeries(out["c3/scores"]), "am"))
    out["c3/weights"] = np.array(C3_WEIGHTS)
    np.savez_compressed(HERE / "golden_configs_v1.npz", **out)
    print("wrote", HERE / "golden_configs_v1.npz", f"({time.time() - t0:.0f} s)")


if __name__ == "__main__":
    main()
