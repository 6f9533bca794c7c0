"""Colorimetric models on the device vs the reference's golden outputs (golden_color_v1.npz).

Tolerances: conversions (BT.709 both ways, luma, hue) are bit-exact; qssim
in the RGB / YCbCr embeddings replays the reference's accumulation order per
window (1e-14, only the final mean's summation order differs); the CIELAB
paths contain a 3x3 matmul the reference runs through BLAS (1e-12); cmssim /
hssim go through the fused SSIM kernels: rect windows on float64 planes use
direct window sums (1e-9), Gaussian windows the fp32 path (1e-5).
"""

import numpy as np
import pytest

import paper_2101_06354_b200 as P
from paper_2101_06354_b200 import errors as E

from test_oracle_color_golden import FRAMES, QSSIM_WINDOWS, frame_case, gcolor  # noqa: F401

pytestmark = pytest.mark.gpu

MAP_WINDOWS = {"r11": P.WindowSpec.rectangular(11), "g15": P.WindowSpec.gaussian(1.5),
               "r7s2": P.WindowSpec.rectangular(7, stride=2)}


def frames(gcolor, name):  # noqa: F811
    h, w, bd, peak, rgb_r, rgb_d, yc_r, yc_d = frame_case(gcolor, name)
    fr = P.ColorFrame(tuple(rgb_r), "rgb", "444", bd)
    fd = P.ColorFrame(tuple(rgb_d), "rgb", "444", bd)
    yr = P.ColorFrame(tuple(yc_r), "ycbcr-bt709", "420", bd)
    yd = P.ColorFrame(tuple(yc_d), "ycbcr-bt709", "420", bd)
    return bd, fr, fd, yr, yd


@pytest.mark.parametrize("name", FRAMES)
def test_conversions_bit_exact(cuda, gcolor, name):  # noqa: F811
    bd, fr, fd, yr, yd = frames(gcolor, name)
    assert np.array_equal(np.stack(P.rgb_to_ycbcr_bt709(fr).channels), gcolor[f"{name}/rgb2ycc"])
    assert np.array_equal(np.stack(P.ycbcr_bt709_to_rgb(yr).channels), gcolor[f"{name}/ycc2rgb"])
    assert np.array_equal(P.luma_of(fr).samples, gcolor[f"{name}/luma"])
    assert np.array_equal(P.hue_plane(fr).samples, gcolor[f"{name}/hue"])
    assert np.allclose(P.delta_e_map(fr, fd), gcolor[f"{name}/de_smooth"], rtol=0, atol=1e-10)
    assert np.allclose(P.delta_e_map(fr, fd, False), gcolor[f"{name}/de_plain"], rtol=0, atol=1e-10)


@pytest.mark.parametrize("name", FRAMES)
def test_qssim(cuda, gcolor, name):  # noqa: F811
    bd, fr, fd, yr, yd = frames(gcolor, name)
    for wname, k, s in QSSIM_WINDOWS:
        win = P.WindowSpec.rectangular(k, stride=s)
        for space in ("rgb", "ycbcr", "lab"):
            got = P.qssim(fr, fd, win, space=space)
            want = float(gcolor[f"{name}/qssim/{space}/{wname}"])
            assert abs(got - want) < (1e-12 if space == "lab" else 1e-14), (space, wname, got, want)
        got = P.qssim(yr, yd, win, space="ycbcr")
        assert abs(got - float(gcolor[f"{name}/qssim_ycc420/{wname}"])) < 1e-14
    assert P.qssim(fr, fr) == pytest.approx(1.0, abs=1e-12)
    with pytest.raises(E.ValidationError):
        P.qssim(fr, fd, P.WindowSpec.gaussian(1.5))
    with pytest.raises(E.WrongSpace):
        P.qssim(yr, yd, space="rgb")


@pytest.mark.parametrize("name", FRAMES)
def test_cmssim_hssim(cuda, gcolor, name):  # noqa: F811
    bd, fr, fd, yr, yd = frames(gcolor, name)
    for wname, win in MAP_WINDOWS.items():
        tol = 1e-5 if win.shape == "gauss" else 1e-9
        cfg = P.SsimConfig(bit_depth=bd, window=win)
        for tag, (a, b) in (("", (fr, fd)), ("_ycc", (yr, yd))):
            got = P.cmssim(a, b, win, cfg)
            assert abs(got - float(gcolor[f"{name}/cmssim{tag}/{wname}"])) < tol, (tag, wname)
            got = P.hssim(a, b, win, cfg)
            assert abs(got - float(gcolor[f"{name}/hssim{tag}/{wname}"])) < tol, (tag, wname)
    assert P.cmssim(fr, fr) == pytest.approx(1.0, abs=1e-12)
    assert P.hssim(fr, fr) == pytest.approx(1.0, abs=1e-12)


@pytest.mark.parametrize("name", FRAMES)
def test_score_frame_pair_color_models(cuda, gcolor, name):  # noqa: F811
    bd, fr, fd, yr, yd = frames(gcolor, name)
    for model, space in (("qssim", "rgb"), ("qssim", "ycbcr"), ("qssim", "lab"), ("cmssim", "rgb"),
                         ("hssim", "rgb")):
        cfg = P.SsimConfig(bit_depth=bd, color=P.ColorModelSpec(model, space=space))
        for tag, (a, b) in (("rgb", (fr, fd)), ("ycc", (yr, yd))):
            rec = P.score_frame_pair(a, b, cfg)
            want = float(gcolor[f"{name}/frame/{model}_{space}/{tag}"])
            assert abs(rec.score - want) < 1e-9, (model, space, tag, rec.score, want)
            assert rec.am is None
