"""Pin the oracle's pooling / adaptation / frame-record restatements to the reference's outputs.

Golden vectors: tests/golden/golden_pool_v1.npz, made by running ssimkit itself
(tests/golden/make_golden_pool.py).  The package's scale-factor arithmetic is
host code and is checked here too.
"""

from pathlib import Path

import numpy as np
import pytest

GOLDEN_POOL = Path(__file__).resolve().parent / "golden" / "golden_pool_v1.npz"

SELECTORS = ("am", "cov", "md", "md:p=3,o=2", "md:p=1,o=0.5", "fns", "dw", "dw:p=2.5", "mink", "mink:p=3",
             "pp", "pp:ps=6,rs=4", "pp:ps=37.5,rs=1000", "pp:ps=100,rs=2", "pp:ps=0,rs=5",
             "lw:a=10,b=5", "lw:a=60,b=0")
MAPS = ("ssimlike", "ties", "wide", "tall", "ones", "single", "pair", "big")
FRAME_CASES = ("enh_1080", "enh_720", "enh_576_10b", "legacy_gauss_fns", "rect_pp", "gauss_md", "rect_lw", "gauss_dw")


@pytest.fixture(scope="session")
def gpool():
    with np.load(GOLDEN_POOL) as z:
        return {k: z[k] for k in z.files}


def big_map():
    """Same recipe as make_golden_pool.big_map (seed 4343)."""
    rng = np.random.default_rng(4343)
    v = np.clip(1.0 - np.abs(rng.standard_cauchy((700, 900))) * 0.01, -1.0, 1.0)
    return v, rng.uniform(0.0, 120.0, v.shape)


def pool_map(gpool, name):
    if name == "big":
        return big_map()
    return gpool[f"pool/{name}/values"], gpool[f"pool/{name}/luma"]


def oracle_params(sel: str) -> tuple[str, dict]:
    from paper_2101_06354_b200.pooling import parse_spatial

    p = parse_spatial(sel)
    return p.kind, dict(p=p.p, o=p.o, a=p.a, b=p.b, ps=p.ps, rs=p.rs)


def frame_inputs(h, w, bd, seed):
    from paper_2101_06354_b200 import synth

    rng = np.random.default_rng(seed)
    peak = float((1 << bd) - 1)
    dt = np.uint8 if bd == 8 else np.uint16
    a = synth.inv_f_noise(rng, h, w, peak).astype(dt)
    amp = 12 * (1 << (bd - 8))
    b = np.clip(a.astype(np.int64) + rng.integers(-amp, amp + 1, a.shape), 0, int(peak)).astype(dt)
    return a, b


# (shape, k, stride, sigma, engine, pool selector, scale policy) of each frame case
FRAME_SPECS = {
    "enh_1080": ("rect", 11, 5, None, "integral", "cov", "dh"),
    "enh_720": ("rect", 11, 5, None, "integral", "cov", "dh"),
    "enh_576_10b": ("rect", 11, 5, None, "integral", "cov", "dh"),
    "legacy_gauss_fns": ("gauss", 11, 1, 1.5, "auto", "fns", "legacy"),
    "rect_pp": ("rect", 11, 1, None, "auto", "pp:ps=10,rs=4", "none"),
    "gauss_md": ("gauss", 11, 1, 1.5, "auto", "md:p=2,o=1", "none"),
    "rect_lw": ("rect", 11, 1, None, "auto", "lw:a=40,b=20", "none"),
    "gauss_dw": ("gauss", 11, 1, 1.5, "auto", "dw:p=2", "none"),
}


@pytest.mark.parametrize("name", MAPS)
def test_oracle_pooling_bit_exact(gpool, oracle, name):
    v, luma = pool_map(gpool, name)
    for sel in SELECTORS:
        kind, params = oracle_params(sel)
        got = oracle.pool_spatial(v, kind, ref_luma=luma, **params)
        assert got == float(gpool[f"pool/{name}/{sel}"]), (name, sel)


def test_oracle_box_downsample_bit_exact(gpool, oracle):
    for name in ("u8", "u16", "even", "f64", "f64big"):
        a = gpool[f"down/{name}/in"]
        for f in (1, 2, 3, 4, 5, 6, 7, 9, 12, 17):
            got = np.asarray(oracle.box_downsample(a, f), dtype=np.float64)
            assert np.array_equal(got, gpool[f"down/{name}/f{f}"]), (name, f)


def test_scale_factor_table(gpool, oracle):
    import paper_2101_06354_b200 as P

    sizes = ((176, 144), (352, 288), (640, 480), (720, 576), (1280, 720), (1920, 1080), (2560, 1440),
             (3840, 2160), (300, 200), (383, 1000))
    policies = (P.ScalePolicy.none(), P.ScalePolicy.legacy256(), P.ScalePolicy.legacy256("ceil"),
                P.ScalePolicy.enhanced_dh(3.0), P.ScalePolicy.enhanced_dh(1.5), P.ScalePolicy.enhanced_dh(6.0),
                P.ScalePolicy.sast(1000.0), P.ScalePolicy.sast(2500.0, 30.0, 45.0))
    table = gpool["factor/table"]
    for i, (w, h) in enumerate(sizes):
        for j, pol in enumerate(policies):
            assert P.policy_factor(pol, w, h) == table[i, j], (w, h, pol)
            kw = dict(rounding=pol.rounding, d_over_h=pol.d_over_h, distance=pol.distance, theta_h=pol.theta_h,
                      theta_w=pol.theta_w)
            assert oracle.scale_factor(pol.kind, w, h, **kw) == table[i, j]
    assert P.round_half_away(2.5) == 3 and P.round_half_away(-2.5) == -3 and P.round_half_away(4.49) == 4


@pytest.mark.parametrize("name", FRAME_CASES)
def test_oracle_frame_record(gpool, oracle, name):
    seed, h, w, bd = (int(x) for x in gpool[f"frame/{name}/seed"])
    a, b = frame_inputs(h, w, bd, seed)
    shape, k, stride, sigma, engine, sel, policy = FRAME_SPECS[name]
    factor = oracle.scale_factor(policy, w, h)
    kind, params = oracle_params(sel)
    got = oracle.luma_frame_record(a, b, shape=shape, k=k, stride=stride, sigma=sigma, bit_depth=bd,
                                   engine=engine, factor=factor, pool=kind, **params)
    want = gpool[f"frame/{name}/record"]
    assert np.array_equal(np.array(got), want), (got, want)


def test_pipeline_presets_host_logic():
    import paper_2101_06354_b200 as P
    from paper_2101_06354_b200 import errors as E

    enh = P.expand_preset("enhanced").config
    assert enh.window == P.WindowSpec.rectangular(11, stride=5) and enh.engine == "integral"
    assert enh.scaling == P.ScalePolicy.enhanced_dh(3.0) and enh.spatial_pool == "cov"
    assert P.expand_preset("default").config == P.SsimConfig()
    with pytest.raises(E.ValidationError):
        P.expand_preset("fast")
    with pytest.raises(E.ValidationError):
        P.PipelineSpec(kt=2, config=P.SsimConfig(window=P.WindowSpec.gaussian(1.5)))
    assert P.policy_factor(enh.scaling, 1920, 1080) == 4
