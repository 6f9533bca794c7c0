"""GPU parity at the BASELINE.json configurations' stated sizes, against scores the REFERENCE produced.

``tests/golden/golden_configs_v1.npz`` holds the reference's (ssimkit's) own per-frame
scores for every frame of configs 2 and 3, four config-4 pairs and eight config-5 pairs
(script: ``tests/golden/make_golden_configs.py``).  The frames are regenerated here from
``synth``'s seeds; each frame's CRC32 is checked first, so a changed synthetic input
fails as such and never as an engine mismatch.

Tolerances (north star): per-frame SSIM / MS-SSIM scores within 1e-5 absolute of the
float64 reference for the fp32 Gaussian path; the rect/integral path (exact integer
sums, float64 epilogue) within 1e-12.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import zlib
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np
import pytest

import paper_2101_06354_b200 as P
from paper_2101_06354_b200 import engine, synth

pytestmark = pytest.mark.gpu

SCORE_TOL = 1e-5
EXACT_TOL = 1e-12
GOLDEN = Path(__file__).resolve().parent / "golden" / "golden_configs_v1.npz"


@pytest.fixture(scope="module")
def gold():
    with np.load(GOLDEN) as z:
        return {k: z[k] for k in z.files}


def _crc(*arrays) -> int:
    c = 0
    for a in arrays:
        c = zlib.crc32(np.ascontiguousarray(a).tobytes(), c)
    return c


def _pool():
    # spawn: the parent already holds a CUDA context, which fork would copy
    return ProcessPoolExecutor(min(8, os.cpu_count() or 1), mp_context=mp.get_context("spawn"))


def _dct_pair(args):
    return synth.dct_pair(*args)


def _c3_frames(idx):
    vid = synth.VideoConfig3()
    return [vid.pair(t) for t in idx]


def _check_inputs(pairs, crcs, tag):
    got = np.array([_crc(*p) for p in pairs], np.uint32)
    bad = np.flatnonzero(got != crcs)
    assert bad.size == 0, f"{tag}: regenerated synthetic inputs differ from the golden's at frames {bad[:8]}"


def _dct_batch(cfgno, n, h, w):
    import torch

    with _pool() as ex:
        pairs = list(ex.map(_dct_pair, [(cfgno, i, h, w) for i in range(n)]))
    ref = torch.from_numpy(np.stack([p[0] for p in pairs]))
    dist = torch.from_numpy(np.stack([p[1] for p in pairs]))
    return pairs, ref, dist


def _gauss():
    return P.SsimConfig(window=P.WindowSpec.gaussian(1.5))


def _device_msssim(ref, dist, cfg, levels, cuda):
    r, d = ref.to(cuda), dist.to(cuda)
    ms, terms = P.msssim_batch(r, d, cfg, P.MultiscaleSpec.product(levels), with_ssim=True)
    pair = engine.device_pair(r, d, cfg.bit_depth, cfg.window.shape == "gauss")
    lv, _, _ = engine.msssim_levels(pair, cfg.window, cfg.c1, cfg.c2, levels)
    t = np.stack([terms.score.cpu().numpy(), terms.l_mean.cpu().numpy(), terms.cs_mean.cpu().numpy()], axis=1)
    return ms.cpu().numpy(), t, lv.cpu().numpy()


def test_config2_all_64_pairs(cuda, gold):
    """Config 2 at stated size: 64 x 1080p u8, Gaussian 11/1.5 SSIM terms, the 5 scale scores
    and 5-scale MS-SSIM for every frame of the batch, device-resident and through the
    host API (HostBatchScorer: pinned host -> H2D -> kernels -> D2H)."""
    pairs, ref, dist = _dct_batch(2, 64, 1080, 1920)
    _check_inputs(pairs, gold["c2/crc"], "config 2")
    cfg = _gauss()
    ms, terms, lv = _device_msssim(ref, dist, cfg, 5, cuda)
    assert np.max(np.abs(ms - gold["c2/msssim"])) < SCORE_TOL
    assert np.max(np.abs(terms - gold["c2/terms"])) < SCORE_TOL
    assert np.max(np.abs(lv - gold["c2/levels"])) < SCORE_TOL
    scorer = P.HostBatchScorer(cfg, P.MultiscaleSpec.product(5), mode="both", chunk=8)
    hms, hss = scorer(ref.pin_memory(), dist.pin_memory())
    assert np.array_equal(hms, ms) and np.array_equal(hss, terms)  # same kernels, same partial order


def test_config2_reference_default_window(cuda, gold):
    """The same 64 pairs under the reference's default window (rect 11, auto engine): exact
    integer sums at scale 0, float64 box sums on the dyadic levels."""
    pairs, ref, dist = _dct_batch(2, 64, 1080, 1920)
    _check_inputs(pairs, gold["c2/crc"], "config 2")
    ms = P.msssim_batch(ref.to(cuda), dist.to(cuda), P.SsimConfig(), P.MultiscaleSpec.product(5))
    assert np.max(np.abs(ms.cpu().numpy() - gold["c2/msssim_rect11"])) < EXACT_TOL


def test_config3_300_frames_yuv420(cuda, gold):
    """Config 3 at stated size: 300 frames of 1080p YUV420, per-plane Gaussian SSIM combined
    with Y:U:V = 4:1:1, then the temporal mean, through SequenceScorer."""
    n = 300
    chunks = [list(range(i, min(n, i + 38))) for i in range(0, n, 38)]
    with _pool() as ex:
        frames = [f for part in ex.map(_c3_frames, chunks) for f in part]
    _check_inputs([(*r, *d) for r, d in frames], gold["c3/crc"], "config 3")
    cfg = _gauss()
    wts = tuple(float(x) for x in gold["c3/weights"])
    res = P.SequenceScorer(cfg, batch_frames=16, color_weights=wts).score([r for r, _ in frames],
                                                                          [d for _, d in frames])
    assert len(res.scores) == n
    assert np.max(np.abs(res.scores - gold["c3/scores"])) < SCORE_TOL
    assert abs(res.pooled - float(gold["c3/pooled"])) < SCORE_TOL
    # per-plane scores (luma at 1080p, chroma at 540x960) for a spread of frames
    import torch

    for t in (0, 1, 149, 299):
        r, d = frames[t]
        for p in range(3):
            s = P.ssim_batch(torch.from_numpy(r[p][None]).to(cuda), torch.from_numpy(d[p][None]).to(cuda), cfg)
            assert abs(float(s[0]) - gold["c3/planes"][t, p]) < SCORE_TOL, (t, p)


def test_config4_4k_10bit_box_scores(cuda, gold):
    """Config 4 pairs at stated size: rect 8 stride 4 integral SSIM on 4K 10-bit (u16)."""
    from paper_2101_06354_b200 import synth as S

    cfg = P.SsimConfig(bit_depth=10, window=P.WindowSpec.rectangular(8, stride=4), engine="integral")
    n = len(gold["c4/crc"])
    pairs = [S.config4_pair(i) for i in range(n)]
    _check_inputs(pairs, gold["c4/crc"], "config 4")
    import torch

    ref = torch.from_numpy(np.stack([p[0] for p in pairs])).to(cuda)
    dist = torch.from_numpy(np.stack([p[1] for p in pairs])).to(cuda)
    t = P.ssim_terms_batch(ref, dist, cfg)
    got = np.stack([t.score.cpu().numpy(), t.l_mean.cpu().numpy(), t.cs_mean.cpu().numpy()], axis=1)
    assert np.max(np.abs(got - gold["c4/terms"])) < EXACT_TOL


def test_config5_4k_ssim_and_msssim(cuda, gold):
    """Config 5 at stated size: 4K u8, Gaussian SSIM terms + 5 scale scores + MS-SSIM per pair
    (the 4K pyramid's level 1 is a 1080x1920 scaled-u16 plane on the coarse-level kernel)."""
    n = len(gold["c5/crc"])
    pairs, ref, dist = _dct_batch(5, n, 2160, 3840)
    _check_inputs(pairs, gold["c5/crc"], "config 5")
    ms, terms, lv = _device_msssim(ref, dist, _gauss(), 5, cuda)
    assert np.max(np.abs(ms - gold["c5/msssim"])) < SCORE_TOL
    assert np.max(np.abs(terms - gold["c5/terms"])) < SCORE_TOL
    assert np.max(np.abs(lv - gold["c5/levels"])) < SCORE_TOL
