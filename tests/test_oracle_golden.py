"""Pin the CPU oracle against the reference's own outputs (golden vectors) and KATs.

The golden vectors were produced by running ssimkit itself
(tests/golden/make_golden.py).  The oracle must reproduce them bit for bit
for integer and float64 work, because every GPU parity test trusts it.
"""

import hashlib
import math

import numpy as np
import pytest

MAP_CASES = {
    # name: window kwargs for the oracle, bit depth
    "gauss11": (dict(shape="gauss", k=11, sigma=1.5), 8),
    "gauss_s3": (dict(shape="gauss", k=11, sigma=1.5, stride=3), 8),
    "gauss13_10b": (dict(shape="gauss", k=13, sigma=2.0), 10),
    "rect11": (dict(shape="rect", k=11), 8),
    "rect8s4_10b": (dict(shape="rect", k=8, stride=4, engine="integral"), 10),
    "rect11_16b": (dict(shape="rect", k=11), 16),
    "rect1": (dict(shape="rect", k=1, engine="naive"), 8),
    "rect16": (dict(shape="rect", k=16, engine="naive"), 8),
    "rect5_float": (dict(shape="rect", k=5), 8),
}


@pytest.mark.parametrize("name", sorted(MAP_CASES))
def test_maps_and_stats_bit_exact(golden, oracle, name):
    win, bd = MAP_CASES[name]
    a, b = golden[f"{name}/ref"], golden[f"{name}/dist"]
    l_map, cs_map, q = oracle.ssim_maps(a, b, bit_depth=bd, **win)
    assert np.array_equal(l_map, golden[f"{name}/l"])
    assert np.array_equal(cs_map, golden[f"{name}/cs"])
    assert np.array_equal(q, golden[f"{name}/q"])
    st = np.stack(oracle.local_statistics(a, b, **win))
    assert np.array_equal(st, golden[f"{name}/stats"])
    assert float(q.mean()) == float(golden[f"{name}/score"])


@pytest.mark.parametrize("name,k,s", [("rect8s4_10b", 8, 4), ("rect11_16b", 11, 1)])
def test_integer_window_sums_exact(golden, oracle, name, k, s):
    got = oracle.box_window_sums(golden[f"{name}/ref"], golden[f"{name}/dist"], k, s)
    assert got.dtype == np.int64
    assert np.array_equal(got, golden[f"{name}/wsums"])


def test_sat_and_downsample(golden, oracle):
    iset = oracle.integral_set(golden["sat/ref"], golden["sat/dist"])
    assert np.array_equal(np.stack([iset[t] for t in oracle.TABLES]), golden["sat/tables"])
    assert np.array_equal(oracle.dyadic_downsample(golden["down/in"]), golden["down/out"])


def test_multiscale(golden, oracle):
    a, b = golden["ms_gauss/ref"], golden["ms_gauss/dist"]
    win = dict(shape="gauss", k=11, sigma=1.5)
    levels = oracle.scale_scores(a, b, 5, **win)
    assert levels == list(golden["ms_gauss/levels"])
    assert oracle.combine_scale_scores(levels) == float(golden["ms_gauss/score"])
    a, b = golden["ms_rect5/ref"], golden["ms_rect5/dist"]
    win = dict(shape="rect", k=5)
    assert oracle.scale_scores(a, b, 4, **win) == list(golden["ms_rect5/levels4"])
    assert oracle.msssim(a, b, 3, "sum", (0.2, 0.3, 0.5), **win) == float(golden["ms_rect5/sum3"])
    assert oracle.msssim(a, b, 4, "fast4", None, **win) == float(golden["ms_rect5/fast4"])


def test_color_and_temporal(golden, oracle):
    ref = [golden[f"color/ref{i}"] for i in range(3)]
    dist = [golden[f"color/dist{i}"] for i in range(3)]
    win = dict(shape="gauss", k=11, sigma=1.5)
    scores = oracle.channel_scores(ref, dist, **win)
    assert np.array_equal(np.array(scores), golden["color/per_plane"])
    assert oracle.fixed_weight(scores, (4 / 6, 1 / 6, 1 / 6)) == float(golden["color/fixed"])
    assert oracle.channelwise(scores, -0.3, -0.3) == float(golden["color/cw"])
    assert oracle.pool_temporal_am(golden["temporal/series"]) == float(golden["temporal/am"])


def test_config1_generator_and_score(golden, oracle):
    from paper_2101_06354_b200 import synth

    a, b = synth.config1_pair()
    digest = np.frombuffer(hashlib.sha256(a.tobytes() + b.tobytes()).digest(), dtype=np.uint8)
    assert np.array_equal(digest, golden["config1/sha256"]), "seeded generator drifted"
    terms = oracle.ssim_terms(a, b, shape="gauss", k=11, sigma=1.5)
    assert np.array_equal(np.array(terms), golden["config1/terms"])


# --- known-answer values quoted by the reference's tests ---

def test_kat_gaussian_centre_weight(oracle):
    # tests/test_stats.py:60
    assert oracle.gaussian_kernel(1.5, 11)[5, 5] == pytest.approx(0.07076223776394697, abs=1e-15)
    z = sum(math.exp(-(i * i + j * j) / 4.5) for i in range(-5, 6) for j in range(-5, 6))
    assert oracle.gaussian_kernel(1.5)[5, 5] == pytest.approx(1.0 / z, abs=1e-15)


def test_kat_constant_pair(oracle):
    # tests/test_ssim.py:20, :31-37
    a = np.full((20, 20), 100, dtype=np.uint8)
    b = np.full((20, 20), 110, dtype=np.uint8)
    l_map, cs_map, q = oracle.ssim_maps(a, b)
    assert np.allclose(l_map, 0.9954764440915066, atol=1e-12)
    assert np.allclose(cs_map, 1.0, atol=1e-12)


def test_kat_small_tables(oracle):
    # tests/test_stats.py:94-97 and tests/test_multiscale.py:21-25
    a = np.array([[1, 2], [3, 4]], dtype=np.uint8)
    assert oracle.integral_set(a, a)["sum1"][2, 2] == 10
    assert oracle.dyadic_downsample(a)[0, 0] == 2.5


def test_grid_shape_formula(oracle, rng):
    # tests/test_stats.py:229-234
    a = rng.integers(0, 256, (37, 23)).astype(np.uint8)
    for k, s in [(5, 1), (5, 3), (8, 4), (11, 5)]:
        mu1 = oracle.local_statistics(a, a, "rect", k, s)[0]
        assert mu1.shape == ((37 - k) // s + 1, (23 - k) // s + 1)


def test_ssim3d_oracle_against_golden(golden, oracle):
    fa = [golden[f"vol/ref{i}"] for i in range(7)]
    fb = [golden[f"vol/dist{i}"] for i in range(7)]
    assert oracle.ssim3d_series(fa, fb, 3, k=7) == list(golden["vol/series_k3"])
    assert oracle.ssim3d_series(fa, fb, 1, k=5, stride=2) == list(golden["vol/series_k1"])
    vol = oracle.RollingSums(4)
    for a, b in zip(fa, fb):
        vol.push(a, b)
    assert np.array_equal(np.stack(vol.stats(6)), golden["vol/stats_k4_w6"])
    c1, c2 = oracle.constants(8)
    assert np.array_equal(oracle.term_maps(*vol.stats(6), c1, c2)[2], golden["vol/q_k4_w6"])
    fl_a = [f.astype(np.float64) / 3.0 for f in fa]
    fl_b = [f.astype(np.float64) / 3.0 for f in fb]
    assert oracle.ssim3d_series(fl_a, fl_b, 3, k=5, refresh_interval=4) == list(golden["vol/series_float_refresh4"])
    ma = [golden[f"vol/msref{i}"] for i in range(4)]
    mb = [golden[f"vol/msdist{i}"] for i in range(4)]
    assert oracle.msssim3d(ma, mb, 2, levels=3, k=5) == list(golden["vol/ms3d"])
