"""Seeded randomized parity sweep over window shapes, sizes, strides and sample types.

Covers the kernel variants selected by geometry (running-sum vs bulk block-sum rect
kernels, their exact-map and score-only epilogues, classic vs wide-strip Gaussian
kernels with the fused level-1 pyramid) against the oracle.  Rect maps must be
bit-identical, Gaussian maps within 1e-4 and scores within 1e-5.
"""

import numpy as np
import pytest

import paper_2101_06354_b200 as P

pytestmark = pytest.mark.gpu


def _pair(rng, h, w, bd):
    dt = np.uint8 if bd == 8 else np.uint16
    peak = (1 << bd) - 1
    a = rng.integers(0, peak + 1, (h, w)).astype(dt)
    noise = rng.integers(-(peak // 8), peak // 8 + 1, (h, w))
    b = np.clip(a.astype(np.int64) + noise, 0, peak).astype(dt)
    return a, b


def test_rect_fuzz(cuda, oracle):
    rng = np.random.default_rng(91)
    for _ in range(60):
        k = int(rng.integers(1, 17))
        s = int(rng.integers(1, 6))
        bd = int(rng.choice([8, 10]))
        h, w = int(rng.integers(k, 90)), int(rng.integers(k, 140))
        a, b = _pair(rng, h, w, bd)
        cfg = P.SsimConfig(bit_depth=bd, window=P.WindowSpec.rectangular(k, stride=s))
        la, lb = P.LumaPlane(a, bd), P.LumaPlane(b, bd)
        l_map, cs_map, q = oracle.ssim_maps(a, b, shape="rect", k=k, stride=s, bit_depth=bd)
        maps = P.ssim_map(la, lb, cfg)
        assert np.array_equal(maps.q_map.values, q), (k, s, bd, h, w)
        assert np.array_equal(maps.cs_map.values, cs_map)
        terms = P.ssim_terms(la, lb, cfg)  # score-only epilogue
        assert abs(terms[0] - float(q.mean())) < 1e-12 and abs(terms[2] - float(cs_map.mean())) < 1e-12
        rec = P.score_frame_pair(la, lb, P.SsimConfig(bit_depth=bd, window=cfg.window, spatial_pool="cov"))
        assert rec.score == pytest.approx(float(q.std() / q.mean()), rel=1e-9, abs=1e-12)


def test_gauss_fuzz(cuda, oracle):
    rng = np.random.default_rng(92)
    for _ in range(25):
        k = int(rng.choice([3, 5, 7, 9, 11, 13, 15, 17]))
        sigma = float(rng.uniform(0.5, 3.0))
        s = int(rng.integers(1, 4))
        bd = int(rng.choice([8, 10]))
        h, w = int(rng.integers(k, 70)), int(rng.integers(k, 110))
        a, b = _pair(rng, h, w, bd)
        cfg = P.SsimConfig(bit_depth=bd, window=P.WindowSpec.gaussian(sigma, k=k, stride=s))
        win = dict(shape="gauss", k=k, sigma=sigma, stride=s, bit_depth=bd)
        l_map, cs_map, q = oracle.ssim_maps(a, b, **win)
        maps = P.ssim_map(P.LumaPlane(a, bd), P.LumaPlane(b, bd), cfg)
        assert np.max(np.abs(maps.q_map.values - q)) < 1e-4, (k, sigma, s, bd, h, w)
        assert abs(P.ssim_score(P.LumaPlane(a, bd), P.LumaPlane(b, bd), cfg) - float(q.mean())) < 1e-5


def test_msssim_fuzz_wide_and_classic(cuda, oracle):
    """Frames wide enough for the wide-strip + fused level-1 path (w - k + 1 >= 480) and narrow ones."""
    rng = np.random.default_rng(93)
    for h, w, k, levels in ((130, 620, 7, 3), (100, 500, 5, 2), (90, 300, 11, 2), (260, 777, 9, 4)):
        a, b = _pair(rng, h, w, 8)
        cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.2, k=k))
        got = P.scale_scores(a, b, cfg, levels)
        want = oracle.scale_scores(a, b, levels, shape="gauss", k=k, sigma=1.2)
        assert np.max(np.abs(np.array(got) - np.array(want))) < 1e-5, (h, w, k, levels)
        rect = P.SsimConfig(window=P.WindowSpec.rectangular(k))
        got = P.scale_scores(a, b, rect, levels)
        want = oracle.scale_scores(a, b, levels, shape="rect", k=k)
        assert np.max(np.abs(np.array(got) - np.array(want))) < 1e-12


def test_strided_gauss_fuzz(cuda, oracle):
    """Anchor-only strided Gaussian scores (K1s for s = 2..8, K1 masking above) over random
    geometries, window sizes, strides and 8/10-bit samples, batches of 1-3 frames."""
    import torch

    rng = np.random.default_rng(313)
    for _ in range(40):
        k = int(rng.choice([3, 5, 7, 9, 11, 13, 15, 21, 31]))
        sigma = float(rng.uniform(0.4, max(0.5, k / 6.0)))
        s = int(rng.integers(2, 11))
        bd = int(rng.choice([8, 10]))
        n = int(rng.integers(1, 4))
        h, w = int(rng.integers(k, 260)), int(rng.integers(k, 700))
        pairs = [_pair(rng, h, w, bd) for _ in range(n)]
        cfg = P.SsimConfig(bit_depth=bd, window=P.WindowSpec.gaussian(sigma, k=k, stride=s))
        ref = torch.from_numpy(np.stack([p[0] for p in pairs])).cuda()
        dist = torch.from_numpy(np.stack([p[1] for p in pairs])).cuda()
        t = P.ssim_terms_batch(ref, dist, cfg)
        got = np.stack([t.score.cpu().numpy(), t.l_mean.cpu().numpy(), t.cs_mean.cpu().numpy()], axis=1)
        for i, (a, b) in enumerate(pairs):
            want = oracle.ssim_terms(a, b, shape="gauss", k=k, sigma=sigma, stride=s, bit_depth=bd)
            assert np.max(np.abs(got[i] - np.array(want))) < 1e-5, (k, sigma, s, bd, n, h, w, i)
