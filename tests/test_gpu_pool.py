"""Device spatial pooling, resolution adaptation and the per-frame pipeline record vs the reference.

Everything here runs through libssimk.so (ssk_pool_spatial, ssk_box_downsample,
ssk_ssim, ssk_msssim) and is compared with the reference's golden outputs
(tests/golden/golden_pool_v1.npz) and the pinned oracle.

Tolerances: order statistics and box downsampling are exact (bit-equal);
pooled sums differ from numpy's pairwise summation only in float64 rounding
(rel 1e-12); frame records through the fp32 Gaussian path 1e-5 (scores), the
integer rect path 1e-9.
"""

import numpy as np
import pytest

import paper_2101_06354_b200 as P
from paper_2101_06354_b200 import errors as E

from test_oracle_pool_golden import FRAME_CASES, FRAME_SPECS, MAPS, SELECTORS, big_map, frame_inputs, gpool  # noqa: F401

pytestmark = pytest.mark.gpu

EXACT = ("fns",)  # pure order statistics + the same scalar arithmetic


def _close(got, want, sel):
    if sel.split(":")[0] in EXACT:
        return got == want
    return abs(got - want) <= 1e-12 * max(1.0, abs(want))


@pytest.mark.parametrize("name", MAPS)
def test_pool_spatial_vs_reference(cuda, gpool, name):  # noqa: F811
    from test_oracle_pool_golden import pool_map

    v, luma = pool_map(gpool, name)
    for sel in SELECTORS:
        got = P.pool_spatial(v, sel, ref_luma=luma)
        want = float(gpool[f"pool/{name}/{sel}"])
        assert _close(got, want, sel), (name, sel, got, want)


def test_percentiles_exact_random_fp32_and_fp64(cuda):
    import torch

    rng = np.random.default_rng(99)
    for dt in (np.float32, np.float64):
        for shape in ((1, 1), (1, 2), (7, 13), (333, 517), (1070, 1910)):
            v = rng.normal(0.9, 0.05, shape).astype(dt)
            v[rng.random(shape) < 0.2] = dt(1.0)  # heavy ties at 1
            t = torch.from_numpy(v).to(cuda)
            w = v.astype(np.float64)  # fp32 maps pool in float64, like the reference's float64 QualityMap
            for ps in (0.0, 6.0, 25.0, 50.0, 99.9, 100.0):
                got, _ = P.pool_maps(t, f"pp:ps={ps},rs=3")
                want = float(np.where(w <= np.percentile(w, ps), w / 3.0, w).mean()) if ps > 0 else float(w.mean())
                assert abs(float(got[0]) - want) <= 1e-12, (dt, shape, ps)
            got, _ = P.pool_maps(t, "fns")
            q = np.percentile(w, [25.0, 50.0, 75.0])
            assert float(got[0]) == float((w.min() + q[0] + q[1] + q[2] + w.max()) / 5.0), (dt, shape)


def test_pool_maps_batch_equals_single(cuda, oracle):
    import torch

    rng = np.random.default_rng(5)
    maps = rng.uniform(-0.3, 1.0, (6, 41, 57))
    luma = rng.uniform(0.0, 200.0, maps.shape)
    tm, tl = torch.from_numpy(maps).to(cuda), torch.from_numpy(luma).to(cuda)
    for sel in SELECTORS:
        batched, means = P.pool_maps(tm, sel, tl)
        for i in range(6):
            single, _ = P.pool_maps(tm[i], sel, tl[i])
            assert float(batched[i]) == float(single[0])
            # the per-map API reduces in numpy's order (bit-exact to numpy), the batch in a
            # fixed tree order: equal to rounding
            want = P.pool_spatial(maps[i], sel, ref_luma=luma[i])
            assert abs(float(batched[i]) - want) <= 1e-14 * max(1.0, abs(want))
        assert np.allclose(means.cpu().numpy(), maps.reshape(6, -1).mean(axis=1), rtol=1e-14)
    # strided views (a plane of an [n, 3, h, w] map stack) pool in place
    stack = torch.from_numpy(rng.uniform(0, 1, (4, 3, 20, 30))).to(cuda)
    a, _ = P.pool_maps(stack[:, 2], "cov")
    b, _ = P.pool_maps(stack[:, 2].contiguous(), "cov")
    assert torch.equal(a, b)


def test_pool_errors(cuda):
    import torch

    with pytest.raises(E.ZeroMeanCoV):
        P.pool_spatial(np.array([[1.0, -1.0]]), "cov")
    with pytest.raises(E.MissingLumaForLW):
        P.pool_spatial(np.ones((3, 3)), "lw:a=1,b=1")
    with pytest.raises(E.MissingLumaForLW):
        P.pool_spatial(np.ones((3, 3)), "lw", ref_luma=np.ones((2, 2)))
    with pytest.raises(E.EmptyMap):
        P.pool_spatial(np.zeros((0, 4)), "am")
    nan, _ = P.pool_maps(torch.tensor([[1.0, -1.0]], device=cuda, dtype=torch.float64), "cov", strict=False)
    assert torch.isnan(nan).all()


def test_box_downsample_bit_exact(cuda, gpool):
    for name in ("u8", "u16", "even", "f64", "f64big"):
        a = gpool[f"down/{name}/in"]
        for f in (1, 2, 3, 4, 5, 6, 7, 9, 12, 17):
            got = np.asarray(P.box_downsample(a, f), dtype=np.float64)
            assert np.array_equal(got, gpool[f"down/{name}/f{f}"]), (name, f)
    lp = P.LumaPlane(gpool["down/u16/in"], 10)
    out = P.box_downsample(lp, 4)
    assert isinstance(out, P.LumaPlane) and out.bit_depth == 10
    with pytest.raises(E.ValidationError):
        P.box_downsample(gpool["down/u8/in"], 0)


def _config(name, bd):
    shape, k, stride, sigma, engine, sel, policy = FRAME_SPECS[name]
    if name.startswith("enh"):
        return P.expand_preset("enhanced").config.for_bit_depth(bd)
    win = P.WindowSpec.gaussian(1.5) if shape == "gauss" else P.WindowSpec.rectangular(11)
    pol = P.ScalePolicy.legacy256() if policy == "legacy" else P.ScalePolicy.none()
    return P.SsimConfig(bit_depth=bd, window=win, scaling=pol, spatial_pool=sel)


@pytest.mark.parametrize("name", FRAME_CASES)
def test_frame_record_vs_reference(cuda, gpool, name):  # noqa: F811
    seed, h, w, bd = (int(x) for x in gpool[f"frame/{name}/seed"])
    a, b = frame_inputs(h, w, bd, seed)
    cfg = _config(name, bd)
    rec = P.score_frame_pair(P.LumaPlane(a, bd), P.LumaPlane(b, bd), cfg)
    want = gpool[f"frame/{name}/record"]
    got = np.array([rec.score, rec.am, rec.l_mean, rec.cs_mean])
    tol = 1e-5 if cfg.window.shape == "gauss" else 1e-9  # fp32 Gaussian path / exact integer rect path
    assert np.allclose(got, want, rtol=0, atol=tol), (got, want)


def test_enhanced_batch_and_sequence(cuda, gpool):
    import torch

    cfg = P.expand_preset("enhanced").config
    frames = [frame_inputs(1080, 1920, 8, 7001 + 100 * i) for i in range(3)]
    ref = torch.from_numpy(np.stack([f[0] for f in frames])).to(cuda)
    dist = torch.from_numpy(np.stack([f[1] for f in frames])).to(cuda)
    rec = P.score_batch(ref, dist, cfg)
    for i, (a, b) in enumerate(frames):
        single = P.score_frame_pair(a, b, cfg)
        assert float(rec.score[i]) == single.score
        assert float(rec.am[i]) == single.am
    seq = P.SequenceScorer(cfg, batch_frames=2).score([f[0] for f in frames], [f[1] for f in frames])
    assert np.array_equal(seq.scores, rec.score.cpu().numpy())
    assert seq.pooled == pytest.approx(float(rec.score.mean()), abs=1e-15)
    # the golden frame itself through the batch path
    a, b = frame_inputs(1080, 1920, 8, 7001)
    r1 = P.score_batch(torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda), cfg)
    want = gpool["frame/enh_1080/record"]
    assert abs(float(r1.score[0]) - want[0]) <= 1e-12 and abs(float(r1.am[0]) - want[1]) <= 1e-12


def test_scaled_msssim_and_non_pow2_factor(cuda, oracle):
    # legacy rule at 720p -> factor 3 (float block means path); MS-SSIM after scaling
    a, b = frame_inputs(720, 1280, 8, 31)
    cfg = P.SsimConfig(window=P.WindowSpec.rectangular(8), scaling=P.ScalePolicy.legacy256(), spatial_pool="pp:ps=5,rs=8")
    rec = P.score_frame_pair(a, b, cfg)
    want = oracle.luma_frame_record(a, b, shape="rect", k=8, factor=3, pool="pp", ps=5.0, rs=8.0)
    assert np.allclose([rec.score, rec.am, rec.l_mean, rec.cs_mean], want, rtol=0, atol=1e-9)
    ms = P.SsimConfig(window=P.WindowSpec.gaussian(1.5), scaling=P.ScalePolicy.legacy256(),
                      multiscale=P.MultiscaleSpec.product(3))
    got = P.score_frame_pair(a, b, ms).score
    x, y = oracle.box_downsample(a, 3), oracle.box_downsample(b, 3)
    assert got == pytest.approx(oracle.msssim(x, y, 3, shape="gauss", k=11, sigma=1.5), abs=1e-5)
    a, b = frame_inputs(1080, 1920, 8, 32)  # factor 4: exact scaled-integer pyramid input
    got = P.score_frame_pair(a, b, P.SsimConfig(window=P.WindowSpec.rectangular(5), scaling=P.ScalePolicy.legacy256(),
                                                multiscale=P.MultiscaleSpec.product(3))).score
    x, y = oracle.box_downsample(a, 4), oracle.box_downsample(b, 4)
    assert got == pytest.approx(oracle.msssim(x, y, 3, shape="rect", k=5), abs=1e-12)


def test_mssim_pools_on_device(cuda):
    rng = np.random.default_rng(8)
    v = rng.uniform(-0.2, 1.0, (37, 41))
    assert P.mssim(v) == pytest.approx(float(v.mean()), rel=1e-14)
    maps = P.ssim_map(rng.integers(0, 256, (40, 50)).astype(np.uint8), rng.integers(0, 256, (40, 50)).astype(np.uint8))
    assert P.mssim(maps) == pytest.approx(float(maps.q_map.values.mean()), rel=1e-14)
    with pytest.raises(E.EmptyMap):
        P.mssim(np.zeros((0, 3)))


def test_fused_moment_pooling_matches_map_pooling(cuda):
    """CoV / MD(2) from the in-kernel sum of q^2 (no map) equals pooling the returned map."""
    rng = np.random.default_rng(12)
    a = rng.integers(0, 256, (96, 130)).astype(np.uint8)
    b = np.clip(a.astype(int) + rng.integers(-30, 31, a.shape), 0, 255).astype(np.uint8)
    for win in (P.WindowSpec.rectangular(11, stride=5), P.WindowSpec.rectangular(8), P.WindowSpec.rectangular(7, stride=2)):
        for sel in ("cov", "md:p=2,o=1", "md:p=2,o=3"):
            cfg = P.SsimConfig(window=win, spatial_pool=sel)
            fused = P.score_frame_pair(a, b, cfg)
            q = P.ssim_map(a, b, P.SsimConfig(window=win)).q_map
            assert fused.score == pytest.approx(P.pool_spatial(q, sel), rel=1e-10, abs=1e-14), (win, sel)
            assert fused.am == pytest.approx(float(q.values.mean()), abs=1e-14)


POOL_EXACT_CASES = [
    ("am", {}), ("cov", {}), ("md", {"p": 2.0, "o": 3.0}), ("md", {"p": 1.0, "o": 1.0}), ("md", {"p": 3.0, "o": 1.0}),
    ("dw", {"p": 2.0}), ("dw", {"p": 1.0}), ("dw", {"p": 4.0}), ("mink", {"p": 4.0}), ("mink", {"p": 2.0}),
    ("pp", {"ps": 10.0, "rs": 3.0}), ("pp", {"ps": 6.0, "rs": 4000.0}), ("lw", {"a": 40.0, "b": 0.0}),
    ("lw", {"a": 20.0, "b": 50.0}), ("fns", {}),
]


@pytest.mark.parametrize("shape", [(6, 6), (5, 8), (37, 53), (502, 502), (1070, 1910)])
@pytest.mark.parametrize("kind,kw", POOL_EXACT_CASES)
def test_pool_spatial_bit_exact_vs_numpy(cuda, oracle, shape, kind, kw):
    """The per-map pool_spatial (src/pooling.py:202-243) reduces in numpy's pairwise order on
    the device (ssk_pairwise_sum) and finishes with the reference's scalar expressions: equal
    to numpy's value bit for bit (integer exponents through the correctly rounded power)."""
    import paper_2101_06354_b200 as P

    rng = np.random.default_rng(shape[0] * 7919 + shape[1] * 31 + len(kind))
    v = 1.0 - 0.3 * rng.uniform(0, 1, shape) ** 3
    mu = rng.uniform(0.0, 255.0, shape)
    pool = P.SpatialPooler(kind, **kw)
    got = P.pool_spatial(v, pool, ref_luma=mu if kind == "lw" else None)
    want = oracle.pool_spatial(v, kind, ref_luma=mu if kind == "lw" else None, **kw)
    assert got == want, (got, want)
