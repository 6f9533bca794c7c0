"""Pin the oracle's colorimetric restatements (qssim, cmssim, hssim, conversions) to the reference.

Golden vectors: tests/golden/golden_color_v1.npz, made by running ssimkit
itself (tests/golden/make_golden_color.py); inputs are regenerated here from
the stored seeds with the same recipe.
"""

from pathlib import Path

import numpy as np
import pytest

GOLDEN_COLOR = Path(__file__).resolve().parent / "golden" / "golden_color_v1.npz"
FRAMES = ("a", "b", "c")
QSSIM_WINDOWS = (("r11", 11, 1), ("r7s3", 7, 3), ("r8s2", 8, 2))
MAP_WINDOWS = {"r11": dict(shape="rect", k=11), "g15": dict(shape="gauss", k=11, sigma=1.5),
               "r7s2": dict(shape="rect", k=7, stride=2)}


@pytest.fixture(scope="session")
def gcolor():
    with np.load(GOLDEN_COLOR) as z:
        return {k: z[k] for k in z.files}


def color_frames(h, w, bd, seed):
    """Same recipe as make_golden_color.color_frames."""
    from paper_2101_06354_b200 import synth

    rng = np.random.default_rng(seed)
    peak = (1 << bd) - 1
    dt = np.uint8 if bd == 8 else np.uint16

    def chans(hh, ww):
        return [synth.inv_f_noise(rng, hh, ww, float(peak)).astype(dt) for _ in range(3)]

    def distort(cs, amp):
        return [np.clip(c.astype(np.int64) + rng.integers(-amp, amp + 1, c.shape), 0, peak).astype(dt) for c in cs]

    amp = 10 << (bd - 8)
    rgb_r = chans(h, w)
    rgb_d = distort(rgb_r, amp)
    ch, cw = (h + 1) // 2, (w + 1) // 2
    y = synth.inv_f_noise(rng, h, w, float(peak)).astype(dt)
    yc_r = [y] + [synth.inv_f_noise(rng, ch, cw, float(peak)).astype(dt) for _ in range(2)]
    yc_d = distort(yc_r, amp)
    return rgb_r, rgb_d, yc_r, yc_d


def frame_case(gcolor, name):
    seed, h, w, bd = (int(x) for x in gcolor[f"{name}/seed"])
    return (h, w, bd, float((1 << bd) - 1)) + color_frames(h, w, bd, seed)


@pytest.mark.parametrize("name", FRAMES)
def test_conversions_bit_exact(gcolor, oracle, name):
    h, w, bd, peak, rgb_r, rgb_d, yc_r, yc_d = frame_case(gcolor, name)
    assert np.array_equal(np.stack(oracle.rgb_to_ycbcr(rgb_r, peak)), gcolor[f"{name}/rgb2ycc"])
    ycc = oracle.upsample420(yc_r, h, w)
    assert np.array_equal(np.stack(oracle.ycbcr_to_rgb(ycc, peak)), gcolor[f"{name}/ycc2rgb"])
    assert np.array_equal(oracle.luma_rgb(rgb_r), gcolor[f"{name}/luma"])
    assert np.array_equal(oracle.hue(rgb_r, peak), gcolor[f"{name}/hue"])
    assert np.allclose(oracle.delta_e(rgb_r, rgb_d, peak, True), gcolor[f"{name}/de_smooth"], rtol=0, atol=1e-12)
    assert np.allclose(oracle.delta_e(rgb_r, rgb_d, peak, False), gcolor[f"{name}/de_plain"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("name", FRAMES)
def test_qssim(gcolor, oracle, name):
    h, w, bd, peak, rgb_r, rgb_d, yc_r, yc_d = frame_case(gcolor, name)
    for wname, k, s in QSSIM_WINDOWS:
        for space in ("rgb", "ycbcr", "lab"):
            e1 = oracle.qssim_embedding(rgb_r, space, peak)
            e2 = oracle.qssim_embedding(rgb_d, space, peak)
            got = oracle.qssim(e1, e2, k, s, peak)
            want = float(gcolor[f"{name}/qssim/{space}/{wname}"])
            if space == "lab":  # BLAS matmul inside the Lab conversion: not bit-reproducible
                assert abs(got - want) < 1e-12, (space, wname)
            else:
                assert got == want, (space, wname)
        e1 = oracle.qssim_embedding(yc_r, "ycbcr", peak, ycc=True, h=h, w=w)
        e2 = oracle.qssim_embedding(yc_d, "ycbcr", peak, ycc=True, h=h, w=w)
        assert oracle.qssim(e1, e2, k, s, peak) == float(gcolor[f"{name}/qssim_ycc420/{wname}"])


@pytest.mark.parametrize("name", FRAMES)
def test_cmssim_hssim(gcolor, oracle, name):
    h, w, bd, peak, rgb_r, rgb_d, yc_r, yc_d = frame_case(gcolor, name)
    rgb_yr = oracle.ycbcr_to_rgb(oracle.upsample420(yc_r, h, w), peak)
    rgb_yd = oracle.ycbcr_to_rgb(oracle.upsample420(yc_d, h, w), peak)
    for wname, win in MAP_WINDOWS.items():
        for tag, (a, b) in (("", (rgb_r, rgb_d)), ("_ycc", (rgb_yr, rgb_yd))):
            got = oracle.cmssim(a, b, peak, bd, **win)
            assert abs(got - float(gcolor[f"{name}/cmssim{tag}/{wname}"])) < 1e-12, (tag, wname)
            got = oracle.hssim(a, b, peak, bd, **win)
            assert got == float(gcolor[f"{name}/hssim{tag}/{wname}"]), (tag, wname)
