"""The reference's acceptance criteria (tests/test_acceptance.py) run on the GPU engine.

Criteria of the accelerated path: C1 integral/naive equivalence (here: the
device integer path against the float64 oracle, bit-exact), C2 SSIM axioms,
C3 stride consistency, C4 SSIM-3D (tests/test_gpu_parity.py), C6 multiscale,
and the channel-wise part of C7.  Inputs are generated with the reference
tests' own seeds where they exist (tests/test_acceptance.py:46, :75, :96).
"""

import numpy as np
import pytest

import paper_2101_06354_b200 as P

pytestmark = pytest.mark.gpu


def random_plane(rng, h, w, bd=8):
    return rng.integers(0, (1 << bd), (h, w)).astype(np.uint8 if bd == 8 else np.uint16)


def natural(rng, h, w):
    from paper_2101_06354_b200 import synth

    return synth.inv_f_noise(rng, h, w, 255.0).astype(np.uint8)


def test_c1_integer_path_equals_reference_integral_engine(cuda, oracle):
    rng = np.random.default_rng(101)
    checked = 0
    for _ in range(200):
        h, w = int(rng.integers(16, 65)), int(rng.integers(16, 65))
        a, b = random_plane(rng, h, w), random_plane(rng, h, w)
        for k in (3, 8, 11, 16):
            if k > min(h, w):
                continue
            want = oracle.ssim_maps(a, b, shape="rect", k=k, engine="integral")
            for engine in ("integral", "naive"):
                got = P.ssim_map(a, b, P.SsimConfig(window=P.WindowSpec.rectangular(k), engine=engine))
                assert np.array_equal(got.q_map.values, want[2])
                assert np.array_equal(got.cs_map.values, want[1])
        checked += 1
    assert checked == 200


def test_c2_axioms(cuda):
    rng = np.random.default_rng(202)
    for cfg, tol in ((P.SsimConfig(window=P.WindowSpec.rectangular(8)), 1e-12),
                     (P.SsimConfig(window=P.WindowSpec.gaussian(1.5)), 1e-6)):
        for _ in range(40):
            h, w = int(rng.integers(12, 48)), int(rng.integers(12, 48))
            if cfg.window.k > min(h, w):
                continue
            a, b = random_plane(rng, h, w), random_plane(rng, h, w)
            fwd, rev = P.ssim_map(a, b, cfg), P.ssim_map(b, a, cfg)
            assert np.array_equal(fwd.q_map.values, rev.q_map.values)
            assert np.all(np.abs(fwd.q_map.values) <= 1.0 + 1e-6)
            assert abs(P.ssim_score(a, a, cfg) - 1.0) < tol
            if cfg.window.shape == "rect":
                # unique maximum at 1e-9 resolution: the exact integer path (the criterion's
                # rect-8 window); the fp32 Gaussian path resolves ~1e-7 per window instead
                c = a.copy()
                i, j = int(rng.integers(0, h)), int(rng.integers(0, w))
                c[i, j] = c[i, j] + 1 if c[i, j] < 255 else c[i, j] - 1
                assert P.ssim_score(a, c, cfg) < 1.0 - 1e-9


def test_c3_stride_consistency(cuda):
    rng = np.random.default_rng(303)
    for engine, window in (("integral", P.WindowSpec.rectangular(11)), ("naive", P.WindowSpec.gaussian(1.5))):
        for s in (2, 3, 5):
            a, b = random_plane(rng, 56, 48), random_plane(rng, 56, 48)
            dense = P.local_statistics(a, b, window, engine)
            strided = P.local_statistics(a, b, window.with_stride(s), engine)
            for name in ("mu1", "mu2", "var1", "var2", "cov"):
                assert np.array_equal(getattr(strided, name), getattr(dense, name)[::s, ::s])
    worst = 0.0
    for seed in range(20):
        r = np.random.default_rng(5000 + seed)
        ref = natural(r, 128, 128)
        noise = r.integers(-14, 15, ref.shape)
        dist = np.clip(ref.astype(int) + noise, 0, 255).astype(np.uint8)
        d1 = P.ssim_score(ref, dist, P.SsimConfig(window=P.WindowSpec.rectangular(11, stride=1)))
        d5 = P.ssim_score(ref, dist, P.SsimConfig(window=P.WindowSpec.rectangular(11, stride=5)))
        worst = max(worst, abs(d5 - d1))
    assert worst < 0.02


def test_c6_multiscale(cuda, oracle):
    rng = np.random.default_rng(606)
    cfg = P.SsimConfig(window=P.WindowSpec.rectangular(5))
    a = natural(rng, 128, 128)
    for spec in (P.MultiscaleSpec.product(3), P.MultiscaleSpec.weighted_sum(3), P.MultiscaleSpec.fast4()):
        assert P.msssim(a, a, cfg, spec) == pytest.approx(1.0, abs=1e-12)
    b = np.clip(a.astype(int) + rng.integers(-16, 17, a.shape), 0, 255).astype(np.uint8)
    exps = (0.2, 0.45, 0.35)
    got = P.msssim(a, b, cfg, P.MultiscaleSpec("product", 3, exps))
    assert got == pytest.approx(oracle.msssim(a, b, 3, "product", exps, shape="rect", k=5), abs=1e-9)
    finest_cs = P.ssim_terms(a, b, cfg)[2]
    tail = P.msssim(P.dyadic_downsample(a), P.dyadic_downsample(b), cfg, P.MultiscaleSpec("product", 2, exps[1:]))
    assert got == pytest.approx(max(finest_cs, 0.0) ** exps[0] * tail, abs=1e-9)


def test_c7_channelwise_models(cuda):
    rng = np.random.default_rng(707)
    chans = tuple(natural(rng, 48, 48) for _ in range(3))
    frame = P.rgb_to_ycbcr_bt709(P.ColorFrame(chans))
    for alpha, beta in ((0.1, 0.1), (-0.3, -0.3), (1.0, 2.0)):
        assert P.channelwise_cssim(frame, frame, alpha, beta) == pytest.approx(1.0, abs=1e-9)
    dist_y = np.clip(frame.channels[0] + rng.normal(0, 6, frame.channels[0].shape), 0, 255)
    dist = P.ColorFrame((dist_y,) + frame.channels[1:], "ycbcr-bt709")
    luma = P.ssim_score(frame.channels[0], dist_y)
    assert P.channelwise_cssim(frame, dist, 0.0, 0.0) == pytest.approx(luma, abs=1e-12)
    assert P.fixed_weight_cssim(frame, dist, (1.0, 0.0, 0.0)) == luma
