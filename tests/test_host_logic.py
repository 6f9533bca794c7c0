"""Host-side logic of the drop-in boundary (no GPU): configuration, containers, pooling, errors."""

import numpy as np
import pytest

import paper_2101_06354_b200 as P
from paper_2101_06354_b200 import errors as E
from paper_2101_06354_b200.pooling import parse_spatial, parse_temporal


class TestConfig:
    def test_defaults_match_reference(self):
        cfg = P.SsimConfig()
        assert cfg.window == P.WindowSpec.rectangular(11)  # src/config.py:246
        assert cfg.engine == "auto" and cfg.bit_depth == 8
        assert cfg.c1 == pytest.approx(6.5025) and cfg.c2 == pytest.approx(58.5225)
        assert cfg.c3 == cfg.c2 / 2
        assert P.SsimConfig(bit_depth=10).c1 == pytest.approx(104.6529)

    def test_json_round_trip_bit_exact(self):
        cfg = P.SsimConfig(k1=0.013, window=P.WindowSpec.gaussian(1.5, stride=2),
                           multiscale=P.MultiscaleSpec.weighted_sum(3),
                           color=P.ColorModelSpec("fixed", weights=(0.6, 0.2, 0.2)))
        assert P.SsimConfig.from_json(cfg.to_json()) == cfg

    def test_window_validation(self):
        assert P.WindowSpec.gaussian(1.5).k == 11
        with pytest.raises(E.ValidationError):
            P.WindowSpec("gauss", 4, 1.0)
        with pytest.raises(E.NonPositiveSigma):
            P.WindowSpec.gaussian(0.0, k=3)
        with pytest.raises(E.ValidationError):
            P.WindowSpec.rectangular(0)
        with pytest.raises(E.ValidationError):
            P.WindowSpec("rect", 5, 1.0)
        with pytest.raises(E.ValidationError):
            P.WindowSpec.rectangular(5, stride=0)
        assert P.WindowSpec.rectangular(8).k == 8  # even rect windows are allowed

    def test_multiscale_spec(self):
        assert P.MultiscaleSpec.product().exponents == P.STANDARD_EXPONENTS
        f4 = P.MultiscaleSpec.fast4().effective_exponents()
        assert sum(f4) == pytest.approx(1.0) and len(f4) == 4
        with pytest.raises(E.ValidationError):
            P.MultiscaleSpec("product", 3, (0.5, 0.5))
        with pytest.raises(E.ValidationError):
            P.MultiscaleSpec("fast4", 5)
        with pytest.raises(E.ValidationError):
            P.MultiscaleSpec.product(6)

    def test_selectors(self):
        assert P.parse_window("rect:8,stride=4") == P.WindowSpec.rectangular(8, stride=4)
        assert P.parse_window("gauss:1.5") == P.WindowSpec.gaussian(1.5)
        assert P.parse_window("gauss:1.5,k=13").k == 13
        assert P.parse_multiscale("product:levels=3").levels == 3
        assert P.parse_color("fixed:0.8,0.1,0.1").weights == (0.8, 0.1, 0.1)
        assert P.parse_color("cw:a=-0.2,b=-0.1").alpha == -0.2
        for sel in ("rect:11", "gauss:1.5,k=11,stride=2"):
            assert P.parse_window(sel).selector() == sel
        with pytest.raises(E.ValidationError):
            P.parse_window("box:3")
        with pytest.raises(E.ValidationError):
            P.SsimConfig(spatial_pool="bogus")

    def test_color_spec_validation(self):
        with pytest.raises(E.ValidationError):
            P.ColorModelSpec("fixed", weights=(0.5, 0.2, 0.2))
        with pytest.raises(E.DegenerateWeights):
            P.ColorModelSpec("cw", alpha=-0.5, beta=-0.5)


class TestContainers:
    def test_luma_plane_range_and_freeze(self):
        p = P.LumaPlane(np.array([[0, 255]], dtype=np.uint8))
        assert not p.samples.flags.writeable
        with pytest.raises(E.ValidationError):
            P.LumaPlane(np.array([[0, 256]]))
        with pytest.raises(E.ValidationError):
            P.LumaPlane(np.array([[1.0, np.nan]]))
        with pytest.raises(E.ValidationError):
            P.LumaPlane(np.zeros((2, 2)), bit_depth=7)
        assert P.LumaPlane(np.array([[1023]], dtype=np.uint16), 10).peak == 1023.0

    def test_color_frame_420_dims(self):
        y = np.zeros((5, 7), dtype=np.uint8)
        c = np.zeros((3, 4), dtype=np.uint8)
        f = P.ColorFrame((y, c, c), "ycbcr-bt709", "420")
        assert f.height == 5 and f.width == 7
        with pytest.raises(E.ValidationError):
            P.ColorFrame((y, y, y), "ycbcr-bt709", "420")

    def test_quality_map_rejects_non_finite(self):
        with pytest.raises(E.ValidationError):
            P.QualityMap(np.array([[np.inf]]))
        assert P.QualityMap(np.array([[0.5, 1.0]])).mean() == 0.75

    def test_pair_validation(self):
        a = np.zeros((4, 4), dtype=np.uint8)
        with pytest.raises(E.DimensionMismatch):
            P.validate_frame_pair(a, np.zeros((4, 5), dtype=np.uint8))
        with pytest.raises(E.BitDepthMismatch):
            P.validate_frame_pair(P.LumaPlane(a, 8), P.LumaPlane(a.astype(np.uint16), 10))

    def test_exception_hierarchy(self):
        assert issubclass(E.ValidationError, ValueError)
        for cls in (E.WindowLargerThanImage, E.TooManyLevels, E.EngineShapeMismatch, E.EmptyMap):
            assert issubclass(cls, P.SsimkitError)


class TestPooling:
    @pytest.mark.gpu
    def test_spatial_known_answers(self, cuda):
        # tests/test_pooling.py style known answers
        v = np.array([[0.25, 0.5], [0.75, 1.0]])
        assert P.pool_spatial(v, "am") == 0.625
        assert P.pool_spatial(v, "mink:p=1") == pytest.approx(1 - 0.625)
        assert P.pool_spatial(v, "pp:ps=6,rs=1") == 0.625
        assert P.pool_spatial(v, "lw:a=0,b=0", ref_luma=np.ones_like(v)) == 0.625
        assert P.pool_spatial(v, "md:p=2,o=1") == pytest.approx(float(v.std()))
        assert P.pool_spatial(np.array([0.1, 0.2, 0.5, 0.8, 0.9]), "fns") == pytest.approx(0.5)
        with pytest.raises(E.MissingLumaForLW):
            P.pool_spatial(v, "lw")
        with pytest.raises(E.EmptyMap):
            P.pool_spatial(np.zeros((0, 3)), "am")

    def test_temporal(self):
        s = np.array([0.9, 0.8, 0.7, 0.6])
        assert P.pool_temporal(s, "am") == pytest.approx(0.75)
        assert P.pool_temporal(s, "hm") <= P.pool_temporal(s, "gm") <= P.pool_temporal(s, "am")
        assert P.pool_temporal(s, "median") == pytest.approx(0.75)
        assert P.pool_temporal(s, "wam:k=2") == pytest.approx(0.75)
        assert P.pool_temporal(P.ScoreSeries(s), parse_temporal("am")) == pytest.approx(0.75)
        with pytest.raises(E.EmptySeries):
            P.pool_temporal(np.array([]), "am")
        with pytest.raises(E.ZeroMeanCoV):
            P.pool_temporal(np.array([1.0, -1.0]), "cov")

    def test_selector_round_trip(self):
        for sel in ("am", "md:p=2,o=3", "lw:a=10,b=5", "pp:ps=6,rs=4"):
            assert parse_spatial(sel).selector() == sel
        assert parse_temporal("wam:k=3").selector() == "wam:k=3"


def test_gaussian_kernel_host_helper():
    k = P.gaussian_kernel(1.5)
    assert k.shape == (11, 11) and abs(k.sum() - 1.0) < 1e-12
    assert k[5, 5] == pytest.approx(0.07076223776394697, abs=1e-15)
    assert P.rect_equivalent(1.5, "same-variance") == 7
    assert P.rect_equivalent(1.5, "same-size") == 11


def test_weber_closed_forms():
    assert P.weber_luminance_term(50.0, 0.1, 0.0) == pytest.approx(0.9954751131221721, abs=1e-15)
    assert P.weber_luminance_term(50.0, 0.0, 0.3) == 1.0
    with pytest.raises(ValueError):
        P.weber_luminance_term(0.0, 0.1, 0.0)


def test_no_cpu_fallback():
    """Scoring without a CUDA device fails loudly instead of computing on the host."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    a = np.zeros((16, 16), dtype=np.uint8)
    with pytest.raises(E.EngineUnavailable):
        P.ssim_score(a, a)
    with pytest.raises(E.EngineUnavailable):
        P.msssim(np.zeros((64, 64), dtype=np.uint8), np.zeros((64, 64), dtype=np.uint8),
                 P.SsimConfig(window=P.WindowSpec.rectangular(3)), P.MultiscaleSpec.product(3))


def test_media_ingest_y4m_and_raw(tmp_path):
    from paper_2101_06354_b200 import errors as E
    from paper_2101_06354_b200 import ingest

    rng = np.random.default_rng(5)
    frames = [(rng.integers(0, 256, (6, 8)).astype(np.uint8), rng.integers(0, 256, (3, 4)).astype(np.uint8),
               rng.integers(0, 256, (3, 4)).astype(np.uint8)) for _ in range(3)]
    p = tmp_path / "a.y4m"
    ingest.write_y4m(p, frames, 8, 6)
    src = ingest.open_y4m(p)
    assert len(src) == 3 and src.header.chroma == "420" and src.header.width == 8
    for i, fr in enumerate(frames):
        for got, want in zip(src.planes(i), fr):
            assert np.array_equal(got, want)
    src.close()
    r = tmp_path / "a.yuv"
    ingest.write_planar_raw(r, [tuple(x.astype(np.uint16) * 4 for x in fr) for fr in frames], bit_depth=10)
    raw = ingest.open_raw(r, 8, 6, bit_depth=10)
    assert len(raw) == 3 and np.array_equal(raw.planes(2)[1], frames[2][1].astype(np.uint16) * 4)
    raw.close()
    with pytest.raises(E.SizeNotMultiple):
        ingest.open_raw(r, 8, 5, bit_depth=10)
    bad = tmp_path / "bad.y4m"
    bad.write_bytes(b"NOTY4M W8 H6\n")
    with pytest.raises(E.BadMagic):
        ingest.open_y4m(bad)
    bad.write_bytes(b"YUV4MPEG2 W8 H6 C411\n")
    with pytest.raises(E.UnsupportedChroma):
        ingest.open_y4m(bad)
    bad.write_bytes(b"YUV4MPEG2 W8 H6\nFRAME\n" + b"\0" * 10)
    with pytest.raises(E.TruncatedFrame):
        ingest.open_y4m(bad)


def test_ssim3d_shard_halo_bounds():
    # contiguous blocks, each preceded by the kt-1 frames its first window needs
    got = [P.shard_with_halo(10, r, 3, 3) for r in range(3)]
    assert got == [(0, 0, 4), (2, 4, 7), (5, 7, 10)]
    assert [P.shard_with_halo(10, r, 3, 1) for r in range(3)] == [(0, 0, 4), (4, 4, 7), (7, 7, 10)]
    with pytest.raises(E.ValidationError):
        P.shard_with_halo(10, 0, 2, 0)


def test_sum_difference_epilogue_algebra_matches_ssim_terms():
    """The 4-moment Gaussian score path (csrc/gauss_ssim.cuh, sd_terms) filters a = x + y - 2c,
    b = x - y - d and their squares: with Sm = E[a], Dm = E[b], Var(a) = s1^2 + s2^2 + 2 s12 and
    Var(b) = s1^2 + s2^2 - 2 s12,
        cs = (Var(a) - Var(b) + 2 C2) / (Var(a) + Var(b) + 2 C2),
        l  = (Su^2 - Dt^2 + 2 C1) / (Su^2 + Dt^2 + 2 C1),  Su = Sm + 2c, Dt = Dm + d.
    In float64 this must reproduce src/ssim.py:34-45 term for term; in float32 Var(b) must not
    cancel when ref and dist differ by a large flat offset once b carries the tile shift d
    (flat 0 vs flat 255 was 6.7e-5 off in cs with d = 0)."""
    rng = np.random.default_rng(12)
    c1, c2 = 6.5025, 58.5225
    mu1, mu2 = rng.uniform(0, 255, 1000), rng.uniform(0, 255, 1000)
    var1, var2 = rng.uniform(0, 500, 1000), rng.uniform(0, 500, 1000)
    cov = rng.uniform(-1, 1, 1000) * np.sqrt(var1 * var2)
    c, d = np.round((mu1 + mu2) / 2), np.round(mu1 - mu2)  # the tile shifts (any values work)
    sm, dm = mu1 + mu2 - 2 * c, mu1 - mu2 - d
    ea = var1 + var2 + 2 * cov + sm * sm + 2 * c2  # E[a^2] + 2 C2 (the filter carries 2 C2)
    eb = var1 + var2 - 2 * cov + dm * dm           # E[b^2]
    va, vb = ea - sm * sm, eb - dm * dm
    cs_new = (va - vb) / (va + vb)
    su, dt = sm + 2 * c, dm + d
    h = su * su + 2 * c1
    l_new = (h - dt * dt) / (h + dt * dt)
    l_ref = (2 * mu1 * mu2 + c1) / (mu1 ** 2 + mu2 ** 2 + c1)
    cs_ref = (2 * cov + c2) / (var1 + var2 + c2)
    assert np.max(np.abs(l_new - l_ref)) < 1e-12 and np.max(np.abs(cs_new - cs_ref)) < 1e-12
    # float32, flat 0 vs flat 255 through 11 fp32 taps: without d the filtered E[b^2] and
    # E[b]^2 (65025 each) cancel to a residue of the tap-sum rounding; with d = -255 both are 0
    f = np.float32
    g = np.exp(-((np.arange(11) - 5.0) ** 2) / (2 * 1.5 ** 2))
    taps = (g / g.sum()).astype(f)

    def filt(v):
        acc = f(0.0)
        for t in taps:
            acc = f(acc + f(t * f(v)))
        return acc

    for d32, tol in ((0.0, None), (-255.0, 0.0)):
        b = f(-255.0 - d32)
        vb32 = f(filt(b * b) - f(filt(b) * filt(b)))
        if tol is not None:
            assert abs(float(vb32)) <= tol
        else:
            assert abs(float(vb32)) < 0.1  # the residue the shift removes (vs 2 C2 = 117)


def test_gaussian_epilogue_algebra_matches_ssim_terms():
    """The fused Gaussian epilogue (csrc/gauss_ssim.cuh, hpass) forms every term from the
    symmetric Sm = m1 + m2, Dq = (m1 - m2)^2 and Su = Sm + 2s of the shifted means
    m = mu - s; in float64 this algebra must reproduce src/ssim.py:34-45 term for term, and
    in float32 it must not cancel in dark windows (the shifted form 2 Pm + 2 s Sm + 2 s^2 + C1
    lost ~3e-4 of l at mu ~ 1)."""
    rng = np.random.default_rng(11)
    s, c1, c2 = 128.0, 6.5025, 58.5225
    mu1, mu2 = rng.uniform(0, 255, 1000), rng.uniform(0, 255, 1000)
    var1, var2 = rng.uniform(0, 500, 1000), rng.uniform(0, 500, 1000)
    cov = rng.uniform(-1, 1, 1000) * np.sqrt(var1 * var2)
    m1, m2 = mu1 - s, mu2 - s
    e_sq = var1 + var2 + m1 * m1 + m2 * m2  # E[x'^2 + y'^2]
    e_xy = cov + m1 * m2
    sm, dq = m1 + m2, (m1 - m2) ** 2
    su = sm + 2 * s
    den2 = (e_sq + c2) - 0.5 * (sm * sm + dq)
    num2 = 2 * (e_xy - m1 * m2) + c2
    h = 0.5 * su * su + c1
    l_new, cs_new = (h - 0.5 * dq) / (h + 0.5 * dq), num2 / den2
    l_ref = (2 * mu1 * mu2 + c1) / (mu1 ** 2 + mu2 ** 2 + c1)
    cs_ref = (2 * cov + c2) / (var1 + var2 + c2)
    assert np.max(np.abs(l_new - l_ref)) < 1e-12 and np.max(np.abs(cs_new - cs_ref)) < 1e-12
    # float32 in a dark window (mu ~ 1): the Su / Dq form stays accurate, the shifted one does not
    f = np.float32
    a, b = f(1.0) - f(s), f(2.0) - f(s)  # m1, m2
    sm32, dq32 = f(a + b), f((a - b) * (a - b))
    su32 = f(sm32 + f(2 * s))
    h32 = f(f(f(0.5) * f(su32 * su32)) + f(c1))
    l32 = f(f(h32 - f(0.5) * dq32) / f(h32 + f(0.5) * dq32))
    l64 = (2 * 1.0 * 2.0 + c1) / (1.0 + 4.0 + c1)
    assert abs(float(l32) - l64) < 1e-6
