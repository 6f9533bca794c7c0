"""GPU parity: the sm_100a kernels (through the C ABI) against golden vectors and the oracle.

Tolerances (north star, BASELINE.json): integer window sums bit-exact; rect
windows on integer samples also give bit-exact maps (float64 epilogue in the
reference's operation order); Gaussian windows run in fp32 with maps within
1e-4 and per-frame scores within 1e-5 absolute of the float64 reference.
"""

import numpy as np
import pytest

import paper_2101_06354_b200 as P
from paper_2101_06354_b200 import engine
from paper_2101_06354_b200.errors import (
    BitDepthMismatch,
    DimensionMismatch,
    EngineShapeMismatch,
    TooManyLevels,
    TooSmall,
    ValidationError,
    WindowLargerThanImage,
)

pytestmark = pytest.mark.gpu

MAP_TOL = 1e-4
SCORE_TOL = 1e-5

CASES = {
    "gauss11": (P.SsimConfig(window=P.WindowSpec.gaussian(1.5)), 8, False),
    "gauss_s3": (P.SsimConfig(window=P.WindowSpec.gaussian(1.5, stride=3)), 8, False),
    "gauss13_10b": (P.SsimConfig(bit_depth=10, window=P.WindowSpec.gaussian(2.0)), 10, False),
    "rect11": (P.SsimConfig(), 8, True),
    "rect8s4_10b": (P.SsimConfig(bit_depth=10, window=P.WindowSpec.rectangular(8, stride=4), engine="integral"), 10, True),
    "rect11_16b": (P.SsimConfig(bit_depth=16), 16, True),
    "rect1": (P.SsimConfig(window=P.WindowSpec.rectangular(1), engine="naive"), 8, True),
    "rect16": (P.SsimConfig(window=P.WindowSpec.rectangular(16), engine="naive"), 8, True),
    "rect5_float": (P.SsimConfig(window=P.WindowSpec.rectangular(5)), 8, False),
}


def planes(golden, name, bd):
    return P.LumaPlane(golden[f"{name}/ref"], bd), P.LumaPlane(golden[f"{name}/dist"], bd)


@pytest.mark.parametrize("name", sorted(CASES))
def test_maps_against_golden(cuda, golden, name):
    cfg, bd, exact = CASES[name]
    a, b = planes(golden, name, bd)
    maps = P.ssim_map(a, b, cfg)
    for key, got in (("l", maps.l_map.values), ("cs", maps.cs_map.values), ("q", maps.q_map.values)):
        want = golden[f"{name}/{key}"]
        assert got.shape == want.shape
        if exact:
            assert np.array_equal(got, want), f"{name}/{key} not bit-exact"
        else:
            assert np.max(np.abs(got - want)) < MAP_TOL, f"{name}/{key}"
    assert abs(P.ssim_score(a, b, cfg) - float(golden[f"{name}/score"])) < SCORE_TOL
    q, lm, cm = P.ssim_terms(a, b, cfg)
    assert np.max(np.abs(np.array([q, lm, cm]) - golden[f"{name}/terms"])) < SCORE_TOL


@pytest.mark.parametrize("name", sorted(CASES))
def test_local_statistics_against_golden(cuda, golden, name):
    cfg, bd, exact = CASES[name]
    a, b = planes(golden, name, bd)
    st = P.local_statistics(a, b, cfg.window, cfg.engine)
    got = np.stack([st.mu1, st.mu2, st.var1, st.var2, st.cov])
    want = golden[f"{name}/stats"]
    if exact:
        assert np.array_equal(got, want)
    else:
        scale = max(1.0, float(np.abs(want).max()))
        assert np.max(np.abs(got - want)) / scale < 1e-5
    assert st.grid_shape == want.shape[1:]
    assert st.stride == cfg.window.stride and st.window_size == cfg.window.k


@pytest.mark.parametrize("name,k,s,bd", [("rect8s4_10b", 8, 4, 10), ("rect11_16b", 11, 1, 16)])
def test_integer_window_sums_bit_exact(cuda, golden, name, k, s, bd):
    pair = engine.upload_pair(golden[f"{name}/ref"], golden[f"{name}/dist"], bd, gauss=False)
    got = engine.window_sums(pair, k, s)[0].cpu().numpy()
    assert np.array_equal(got, golden[f"{name}/wsums"])


def test_integral_set_and_window_sum(cuda, golden):
    iset = P.build_integral_set(P.LumaPlane(golden["sat/ref"]), P.LumaPlane(golden["sat/dist"]))
    got = np.stack([iset.table(t) for t in ("sum1", "sum2", "sq1", "sq2", "prod")])
    assert got.dtype == np.int64 and np.array_equal(got, golden["sat/tables"])
    a = golden["sat/ref"].astype(np.int64)
    assert P.window_sum(iset, "sum1", 1, 1, 3) == a[1:4, 1:4].sum()


def test_dyadic_downsample_exact(cuda, golden):
    out = P.dyadic_downsample(P.LumaPlane(golden["down/in"]))
    assert isinstance(out, P.LumaPlane)
    assert np.array_equal(out.samples, golden["down/out"])
    raw = P.dyadic_downsample(golden["down/in"].astype(np.float64) / 3.0)
    assert np.array_equal(raw, golden["down/out"] / 3.0) or np.max(np.abs(raw - golden["down/out"] / 3.0)) < 1e-13
    with pytest.raises(TooSmall):
        P.dyadic_downsample(np.zeros((1, 8), dtype=np.uint8))


def test_msssim_against_golden(cuda, golden):
    a, b = P.LumaPlane(golden["ms_gauss/ref"]), P.LumaPlane(golden["ms_gauss/dist"])
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    levels = P.scale_scores(a, b, cfg, 5)
    assert np.max(np.abs(np.array(levels) - golden["ms_gauss/levels"])) < SCORE_TOL
    assert abs(P.msssim(a, b, cfg, P.MultiscaleSpec.product(5)) - float(golden["ms_gauss/score"])) < SCORE_TOL
    a, b = P.LumaPlane(golden["ms_rect5/ref"]), P.LumaPlane(golden["ms_rect5/dist"])
    cfg = P.SsimConfig(window=P.WindowSpec.rectangular(5))
    levels = P.scale_scores(a, b, cfg, 4)
    assert np.max(np.abs(np.array(levels) - golden["ms_rect5/levels4"])) < 1e-12  # exact pyramid + fp64
    assert abs(P.msssim(a, b, cfg, P.MultiscaleSpec("sum", 3, (0.2, 0.3, 0.5))) - float(golden["ms_rect5/sum3"])) < 1e-12
    assert abs(P.msssim(a, b, cfg, P.MultiscaleSpec.fast4()) - float(golden["ms_rect5/fast4"])) < 1e-12


def test_color_against_golden(cuda, golden):
    ref = P.ColorFrame(tuple(golden[f"color/ref{i}"] for i in range(3)), "ycbcr-bt709", "420")
    dist = P.ColorFrame(tuple(golden[f"color/dist{i}"] for i in range(3)), "ycbcr-bt709", "420")
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    assert abs(P.fixed_weight_cssim(ref, dist, (4 / 6, 1 / 6, 1 / 6), cfg) - float(golden["color/fixed"])) < SCORE_TOL
    assert abs(P.channelwise_cssim(ref, dist, -0.3, -0.3, cfg) - float(golden["color/cw"])) < SCORE_TOL
    per = np.array(P.channel_scores(ref, dist, cfg))
    assert np.max(np.abs(per - golden["color/per_plane"])) < SCORE_TOL
    # (1, 0, 0) weights reduce to the luma score exactly (tests/test_color.py:109-114): a plane's
    # score is mssim(ssim_map(..)) as in the reference; the fused score path agrees to fp32
    luma = P.mssim(P.ssim_map(ref.channels[0], dist.channels[0], cfg))
    assert P.fixed_weight_cssim(ref, dist, (1.0, 0.0, 0.0), cfg) == luma
    assert abs(P.ssim_score(ref.channels[0], dist.channels[0], cfg) - luma) < SCORE_TOL


def test_config1_score(cuda, golden):
    from paper_2101_06354_b200 import synth

    a, b = synth.config1_pair()
    terms = P.ssim_terms(P.LumaPlane(a), P.LumaPlane(b), P.SsimConfig(window=P.WindowSpec.gaussian(1.5)))
    assert np.max(np.abs(np.array(terms) - golden["config1/terms"])) < SCORE_TOL


# --- properties the reference's tests pin -----------------------------------

@pytest.mark.parametrize("cfg", [P.SsimConfig(), P.SsimConfig(window=P.WindowSpec.gaussian(1.5)),
                                 P.SsimConfig(window=P.WindowSpec.rectangular(8, stride=3))])
def test_symmetry_exact(cuda, rng, cfg):
    a = rng.integers(0, 256, (45, 53)).astype(np.uint8)
    b = np.clip(a.astype(int) + rng.integers(-25, 26, a.shape), 0, 255).astype(np.uint8)
    fwd, rev = P.ssim_map(a, b, cfg), P.ssim_map(b, a, cfg)
    for attr in ("l_map", "cs_map", "q_map"):
        assert np.array_equal(getattr(fwd, attr).values, getattr(rev, attr).values)
    assert P.ssim_score(a, b, cfg) == P.ssim_score(b, a, cfg)


@pytest.mark.parametrize("window", [P.WindowSpec.rectangular(11, stride=5), P.WindowSpec.rectangular(11, stride=3),
                                    P.WindowSpec.gaussian(1.5, stride=4), P.WindowSpec.gaussian(1.5, stride=2),
                                    P.WindowSpec.rectangular(8, stride=4)])
def test_stride_is_exact_subsample(cuda, rng, window):
    a = rng.integers(0, 256, (48, 40)).astype(np.uint8)
    b = rng.integers(0, 256, (48, 40)).astype(np.uint8)
    s = window.stride
    strided = P.local_statistics(a, b, window)
    dense = P.local_statistics(a, b, window.with_stride(1))
    for name in ("mu1", "mu2", "var1", "var2", "cov"):
        assert np.array_equal(getattr(strided, name), getattr(dense, name)[::s, ::s])


@pytest.mark.parametrize("cfg", [P.SsimConfig(), P.SsimConfig(window=P.WindowSpec.gaussian(1.5))])
def test_identity_and_bounds(cuda, rng, cfg):
    a = rng.integers(0, 256, (40, 40)).astype(np.uint8)
    b = rng.integers(0, 256, (40, 40)).astype(np.uint8)
    tol = 1e-12 if cfg.window.shape == "rect" else 1e-6
    assert abs(P.ssim_score(a, a, cfg) - 1.0) < tol
    q = P.ssim_map(a, b, cfg).q_map.values
    assert np.all(np.abs(q) <= 1.0 + 1e-6)
    c = a.copy()
    c[7, 9] = c[7, 9] + 1 if c[7, 9] < 255 else c[7, 9] - 1
    assert P.ssim_score(a, c, cfg) < 1.0 - 1e-9


def test_delta_kernel_reproduces_input(cuda, rng):
    a = rng.integers(0, 256, (12, 12)).astype(np.uint8)
    b = rng.integers(0, 256, (12, 12)).astype(np.uint8)
    st = P.local_statistics(P.LumaPlane(a), P.LumaPlane(b), P.WindowSpec.gaussian(0.01), "naive")
    assert np.array_equal(st.mu1, a[1:-1, 1:-1].astype(float))
    assert np.array_equal(st.mu2, b[1:-1, 1:-1].astype(float))


@pytest.mark.parametrize("h,w,k", [(11, 11, 11), (11, 300, 11), (300, 11, 11), (13, 17, 3), (129, 131, 7),
                                   (257, 130, 11), (5, 5, 1), (64, 129, 15)])
def test_edge_geometries_vs_oracle(cuda, oracle, rng, h, w, k):
    a = rng.integers(0, 256, (h, w)).astype(np.uint8)
    b = np.clip(a.astype(int) + rng.integers(-30, 31, a.shape), 0, 255).astype(np.uint8)
    want = oracle.ssim_maps(a, b, shape="rect", k=k)
    got = P.ssim_map(a, b, P.SsimConfig(window=P.WindowSpec.rectangular(k)))
    assert np.array_equal(got.q_map.values, want[2])
    if k >= 3 and k % 2 == 1:
        want = oracle.ssim_maps(a, b, shape="gauss", k=k, sigma=k / 6.0)
        got = P.ssim_map(a, b, P.SsimConfig(window=P.WindowSpec.gaussian(k / 6.0, k=k)))
        assert np.max(np.abs(got.q_map.values - want[2])) < MAP_TOL


def test_errors_match_reference_classes(cuda, rng):
    a = rng.integers(0, 256, (8, 8)).astype(np.uint8)
    with pytest.raises(WindowLargerThanImage):
        P.ssim_map(a, a)  # rect 11 on 8x8
    with pytest.raises(EngineShapeMismatch):
        P.local_statistics(a, a, P.WindowSpec.gaussian(0.5), "integral")
    with pytest.raises(DimensionMismatch):
        P.ssim_score(a, a[:7])
    with pytest.raises(BitDepthMismatch):
        P.ssim_score(P.LumaPlane(a, 8), P.LumaPlane(a.astype(np.uint16), 10))
    big = rng.integers(0, 256, (32, 32)).astype(np.uint8)
    with pytest.raises(TooManyLevels):
        P.msssim(big, big, P.SsimConfig(window=P.WindowSpec.rectangular(5)), P.MultiscaleSpec.product(4))
    with pytest.raises(ValidationError):
        P.msssim(big, big, P.SsimConfig(window=P.WindowSpec.rectangular(5)), P.MultiscaleSpec.off())
    with pytest.raises(ValidationError):
        P.local_statistics(big, big, P.WindowSpec.rectangular(5), "fast")


# --- batched device API and full-size configurations -------------------------

def test_batch_matches_per_pair(cuda, rng):
    import torch

    n, h, w = 5, 70, 90
    a = rng.integers(0, 256, (n, h, w)).astype(np.uint8)
    b = np.clip(a.astype(int) + rng.integers(-20, 21, a.shape), 0, 255).astype(np.uint8)
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    got = P.ssim_batch(ta, tb, cfg).cpu().numpy()
    want = np.array([P.ssim_score(a[i], b[i], cfg) for i in range(n)])
    assert np.array_equal(got, want)
    ms, terms = P.msssim_batch(ta, tb, cfg, P.MultiscaleSpec.product(2), with_ssim=True)
    assert np.array_equal(terms.score.cpu().numpy(), want)
    want_ms = [P.msssim(a[i], b[i], cfg, P.MultiscaleSpec.product(2)) for i in range(n)]
    assert np.max(np.abs(ms.cpu().numpy() - np.array(want_ms))) < 1e-12
    # determinism: bit-identical on a rerun
    assert np.array_equal(P.ssim_batch(ta, tb, cfg).cpu().numpy(), got)


def test_persistent_wide_kernel_multi_tile_ctas(cuda, rng):
    """41 wide u8 frames = 252 tiles > one CTA per SM: persistent CTAs walk several tiles
    (the V-tile ring and its barriers continue across tiles) and every frame's score is
    bit-identical to scoring that frame alone (a handful of tiles, one per CTA)."""
    import torch

    n, h, w = 41, 512, 600
    a = rng.integers(0, 256, (n, h, w)).astype(np.uint8)
    b = np.clip(a.astype(int) + rng.integers(-30, 31, a.shape), 0, 255).astype(np.uint8)
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    terms = P.ssim_terms_batch(ta, tb, cfg)
    got = torch.stack([terms.score, terms.l_mean, terms.cs_mean], 1).cpu().numpy()
    for i in (0, 1, 20, 39, 40):
        one = P.ssim_terms_batch(ta[i:i + 1], tb[i:i + 1], cfg)
        assert np.array_equal(got[i], np.array([one.score.item(), one.l_mean.item(), one.cs_mean.item()]))
    assert abs(got[40, 0] - P.ssim_score(a[40], b[40], cfg)) == 0.0


def test_workspace_keeps_its_guards(cuda, rng, monkeypatch):
    """Bounds evidence without compute-sanitizer (closed on this pool): every library call gets a
    workspace of exactly the queried size carved out of the middle of a larger, pre-filled
    buffer -- the pyramid levels (fused level-1 stores on ragged strips, 16-byte items; the
    pyramid pass) and the per-CTA partial sums live there and must leave every guard byte on
    both sides untouched, for odd geometries, strided scores and 10-bit frames."""
    import torch
    from paper_2101_06354_b200 import _native as nat

    guard = 8192

    class Guarded:
        def __init__(self):
            self.bufs = []

        def get(self, nbytes, device, stream=None):
            nb = (max(int(nbytes), 256) + 255) // 256 * 256
            buf = torch.full((nb + 2 * guard,), 0xA5, dtype=torch.uint8, device=device)
            self.bufs.append(buf)
            return buf[guard:guard + nb]

    g = Guarded()
    monkeypatch.setattr(nat, "WORKSPACE", g)
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    for n, h, w, levels in ((3, 517, 963, 4), (2, 140, 250, 2), (5, 97, 491, 3)):
        a = rng.integers(0, 256, (n, h, w)).astype(np.uint8)
        b = np.clip(a.astype(int) + rng.integers(-20, 21, a.shape), 0, 255).astype(np.uint8)
        ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        P.msssim_batch(ta, tb, cfg, P.MultiscaleSpec.product(levels), with_ssim=True)
        P.ssim_terms_batch(ta, tb, cfg)
        P.ssim_terms_batch(ta, tb, P.SsimConfig(window=P.WindowSpec.gaussian(1.5, stride=3)))
    a16 = rng.integers(0, 1024, (3, 200, 700)).astype(np.uint16)
    b16 = np.clip(a16.astype(int) + rng.integers(-40, 41, a16.shape), 0, 1023).astype(np.uint16)
    c10 = P.SsimConfig(bit_depth=10, window=P.WindowSpec.gaussian(1.5))
    P.msssim_batch(torch.from_numpy(a16).cuda(), torch.from_numpy(b16).cuda(), c10, P.MultiscaleSpec.product(3))
    torch.cuda.synchronize()
    assert len(g.bufs) >= 10
    for buf in g.bufs:
        assert bool((buf[:guard] == 0xA5).all()) and bool((buf[-guard:] == 0xA5).all())


_WS_CASE = r"""
import sys, numpy as np, torch
import paper_2101_06354_b200 as P
rng = np.random.default_rng(77)
cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
out = {}
for name, (n, h, w) in {"wide": (41, 512, 600), "narrow": (5, 70, 90), "odd": (3, 517, 963)}.items():
    a = rng.integers(0, 256, (n, h, w)).astype(np.uint8)
    b = np.clip(a.astype(int) + rng.integers(-30, 31, a.shape), 0, 255).astype(np.uint8)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    t = P.ssim_terms_batch(ta, tb, cfg)
    out[name + "_terms"] = torch.stack([t.score, t.l_mean, t.cs_mean], 1).cpu().numpy()
    out[name + "_ms"] = P.msssim_batch(ta, tb, cfg, P.MultiscaleSpec.product(2 if h < 100 else 3)).cpu().numpy()
np.savez(sys.argv[1], **out)
"""


def test_warp_specialised_kernels_match_the_default_kernels_bit_for_bit(cuda, tmp_path):
    """Wide u8 frames default to the classic kernel (two CTAs per SM) and narrow ones to the
    classic 128-column kernel; SSK_L0_CLASSIC=0 / SSK_NARROW_WS=1 select the persistent and the
    narrow warp-specialised kernels (read once per process, hence subprocesses).  The
    arithmetic per item is the same code, so scores, terms and MS-SSIM (fused level 1) must be
    bit-identical -- 41 wide frames give the persistent CTAs several tiles each.  A third run
    with SSK_FUSED_L1=0 builds pyramid level 1 in the separate pyramid pass: the fused stores
    (16-byte items, odd sizes, ragged last strip) must produce the same exact integers, hence
    the same MS-SSIM bits."""
    import os
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    results = []
    for i, extra in enumerate(({}, {"SSK_L0_CLASSIC": "0", "SSK_NARROW_WS": "1"}, {"SSK_FUSED_L1": "0"})):
        path = str(tmp_path / f"ws{i}.npz")
        env = dict(os.environ, PYTHONPATH=repo + os.pathsep + os.environ.get("PYTHONPATH", ""), **extra)
        r = subprocess.run([sys.executable, "-c", _WS_CASE, path], env=env, capture_output=True, text=True, cwd=repo)
        assert r.returncode == 0, r.stderr[-2000:]
        with np.load(path) as z:
            results.append({k: z[k] for k in z.files})
    for other in results[1:]:
        for k, v in results[0].items():
            assert np.array_equal(v, other[k]), k


@pytest.mark.parametrize("n", [2, 7, 40])
def test_msssim_side_stream_split_is_bit_identical(cuda, rng, n):
    """Large batches run as sub-batches on side streams (engine.SPLIT_MIN_FRAMES); every
    split gives the same bits as one launch sequence, on the caller's stream order."""
    import torch

    h, w = 96, 200
    a = rng.integers(0, 256, (n, h, w)).astype(np.uint8)
    b = np.clip(a.astype(int) + rng.integers(-25, 26, a.shape), 0, 255).astype(np.uint8)
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    pair = engine.device_pair(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), 8, gauss=True)
    spec = P.MultiscaleSpec.product(3)
    outs = []
    for split in (1, 2, 3):
        means, score, sums = engine.msssim_levels(pair, cfg.window, cfg.c1, cfg.c2, 3, with_ssim=True,
                                                  spec=spec, split=split)
        outs.append([t.cpu().numpy() for t in (means, score, sums)])
    for other in outs[1:]:
        for x, y in zip(outs[0], other):
            assert np.array_equal(x, y)
    # the default (split when n >= SPLIT_MIN_FRAMES) agrees as well, on a user stream
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ms = P.msssim_batch(pair.ref, pair.dist, cfg, spec)
    torch.cuda.synchronize()
    assert np.array_equal(ms.cpu().numpy(), outs[0][1])


def test_full_1080p_gauss_ssim_and_msssim(cuda, oracle):
    from paper_2101_06354_b200 import synth

    a, b = synth.dct_pair(2, 0)
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    win = dict(shape="gauss", k=11, sigma=1.5)
    terms = P.ssim_terms(a, b, cfg)
    assert np.max(np.abs(np.array(terms) - np.array(oracle.ssim_terms(a, b, **win)))) < SCORE_TOL
    got = P.scale_scores(a, b, cfg, 5)
    want = oracle.scale_scores(a, b, 5, **win)
    assert np.max(np.abs(np.array(got) - np.array(want))) < SCORE_TOL
    maps = P.ssim_map(a, b, cfg)
    wl, wcs, wq = oracle.ssim_maps(a, b, **win)
    assert np.max(np.abs(maps.q_map.values - wq)) < MAP_TOL
    assert np.max(np.abs(maps.cs_map.values - wcs)) < MAP_TOL


def test_fused_level1_odd_geometry_and_batch(cuda, oracle):
    """The level-0 kernel writes pyramid level 1 (wide u8 path): odd frame sizes, several
    strips / segments and an odd batch (a lone frame in the last packed pair)."""
    import torch
    from paper_2101_06354_b200 import synth

    rng = np.random.default_rng(4711)
    h, w = 517, 963  # odd: the last input row / column drop out of level 1
    frames = []
    for _ in range(3):
        a = synth.inv_f_noise(rng, h, w, 255.0).astype(np.uint8)
        b = np.clip(a.astype(int) + rng.integers(-20, 21, a.shape), 0, 255).astype(np.uint8)
        frames.append((a, b))
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    spec = P.MultiscaleSpec.product(4)
    ref = torch.from_numpy(np.stack([f[0] for f in frames])).to(cuda)
    dist = torch.from_numpy(np.stack([f[1] for f in frames])).to(cuda)
    got = P.msssim_batch(ref, dist, cfg, spec).cpu().numpy()
    for i, (a, b) in enumerate(frames):
        want = oracle.msssim(a, b, 4, shape="gauss", k=11, sigma=1.5)
        assert abs(got[i] - want) < SCORE_TOL
        lv = P.scale_scores(a, b, cfg, 4)
        assert np.max(np.abs(np.array(lv) - np.array(oracle.scale_scores(a, b, 4, shape="gauss", k=11, sigma=1.5)))) \
            < SCORE_TOL


@pytest.mark.parametrize("k,sigma,levels,h,w", [(7, 1.0, 2, 301, 650), (15, 2.3, 3, 422, 703), (17, 2.7, 3, 480, 996)])
def test_fused_level1_window_sizes(cuda, oracle, k, sigma, levels, h, w):
    """Wide-strip kernel + fused level 1 across window sizes (k <= 17 takes the wide path)."""
    from paper_2101_06354_b200 import synth

    rng = np.random.default_rng(k * 100 + levels)
    a = synth.inv_f_noise(rng, h, w, 255.0).astype(np.uint8)
    b = np.clip(a.astype(int) + rng.integers(-25, 26, a.shape), 0, 255).astype(np.uint8)
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(sigma, k=k))
    win = dict(shape="gauss", k=k, sigma=sigma)
    got = P.scale_scores(a, b, cfg, levels)
    want = oracle.scale_scores(a, b, levels, **win)
    assert np.max(np.abs(np.array(got) - np.array(want))) < SCORE_TOL


def test_full_4k_10bit_box_sums_bit_exact(cuda, oracle):
    from paper_2101_06354_b200 import synth

    a, b = synth.config4_pair(0)
    pair = engine.upload_pair(a, b, 10, gauss=False)
    got = engine.window_sums(pair, 8, 4)[0].cpu().numpy()
    want = oracle.box_window_sums(a, b, 8, 4)
    assert got.shape == (5, 539, 959)
    assert np.array_equal(got, want)
    cfg = P.SsimConfig(bit_depth=10, window=P.WindowSpec.rectangular(8, stride=4), engine="integral")
    q = P.ssim_map(P.LumaPlane(a, 10), P.LumaPlane(b, 10), cfg).q_map.values
    assert np.array_equal(q, oracle.ssim_maps(a, b, shape="rect", k=8, stride=4, bit_depth=10)[2])


def test_video_sequence_yuv420(cuda, oracle):
    from paper_2101_06354_b200 import synth

    vid = synth.VideoConfig3(frames=6, h=64, w=96)
    pairs = [vid.pair(t) for t in range(6)]
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    wts = (4 / 6, 1 / 6, 1 / 6)
    res = P.score_sequence([r for r, _ in pairs], [d for _, d in pairs], cfg, batch_frames=4, color_weights=wts)
    win = dict(shape="gauss", k=11, sigma=1.5)
    want = [oracle.fixed_weight(oracle.channel_scores(r, d, **win), wts) for r, d in pairs]
    assert np.max(np.abs(res.scores - np.array(want))) < SCORE_TOL
    assert abs(res.pooled - oracle.pool_temporal_am(want)) < SCORE_TOL
    # luma records carry (score, am, l_mean, cs_mean)
    luma = P.score_sequence([r[0] for r, _ in pairs], [d[0] for _, d in pairs], cfg, batch_frames=4)
    for rec, (r, d) in zip(luma.records, pairs):
        assert np.max(np.abs(np.array([rec.score, rec.l_mean, rec.cs_mean]) -
                             np.array(oracle.ssim_terms(r[0], d[0], **win)))) < SCORE_TOL


@pytest.mark.parametrize("h,w", [(5, 7), (33, 130), (64, 2000), (17, 1)])
@pytest.mark.parametrize("kind", ["u8", "u16", "f64"])
def test_downsample_shapes_and_dtypes(cuda, oracle, rng, h, w, kind):
    if w < 2:
        with pytest.raises(TooSmall):
            P.dyadic_downsample(np.zeros((h, w), dtype=np.uint8))
        return
    if kind == "u8":
        a = rng.integers(0, 256, (h, w)).astype(np.uint8)
    elif kind == "u16":
        a = rng.integers(0, 1024, (h, w)).astype(np.uint16)
    else:
        a = rng.uniform(0, 255, (h, w))
    want = oracle.dyadic_downsample(a)
    got = P.dyadic_downsample(a)
    assert got.shape == want.shape and np.array_equal(got, want)
    got2 = P.dyadic_downsample(got) if min(got.shape) >= 2 else None
    if got2 is not None:
        assert np.array_equal(got2, oracle.dyadic_downsample(want))


@pytest.mark.parametrize("k,s,bd,h,w", [(8, 4, 10, 70, 300), (8, 4, 8, 64, 517), (4, 2, 8, 33, 65), (12, 4, 10, 50, 260),
                                        (8, 8, 10, 40, 270), (16, 8, 8, 47, 300), (10, 2, 8, 31, 90), (4, 4, 12, 30, 80),
                                        (16, 8, 12, 40, 100)])
def test_block_box_path_bit_exact(cuda, oracle, rng, k, s, bd, h, w):
    """Stride-divides-window rect path (block sums): int64 window sums and maps bit-exact."""
    peak = (1 << bd) - 1
    dt = np.uint8 if bd == 8 else np.uint16
    a = rng.integers(0, peak + 1, (h, w)).astype(dt)
    b = np.clip(a.astype(np.int64) + rng.integers(-40, 41, a.shape), 0, peak).astype(dt)
    pair = engine.upload_pair(a, b, bd, gauss=False)
    got = engine.window_sums(pair, k, s)[0].cpu().numpy()
    assert np.array_equal(got, oracle.box_window_sums(a, b, k, s))
    cfg = P.SsimConfig(bit_depth=bd, window=P.WindowSpec.rectangular(k, stride=s))
    maps = P.ssim_map(P.LumaPlane(a, bd), P.LumaPlane(b, bd), cfg)
    want = oracle.ssim_maps(a, b, shape="rect", k=k, stride=s, bit_depth=bd)
    assert np.array_equal(maps.q_map.values, want[2]) and np.array_equal(maps.l_map.values, want[0])
    assert abs(P.ssim_score(P.LumaPlane(a, bd), P.LumaPlane(b, bd), cfg) - float(want[2].mean())) < 1e-12


# --- deeper pyramid / dtype coverage -----------------------------------------

@pytest.mark.parametrize("bd,levels,window", [
    (10, 5, P.WindowSpec.gaussian(1.5)),   # u16 input, u32 pyramid levels
    (12, 4, P.WindowSpec.rectangular(7)),  # u16 input, exact integer pyramid, fp64 epilogue
    (16, 3, P.WindowSpec.gaussian(1.0)),   # full 16-bit range
    (8, 5, P.WindowSpec.gaussian(1.5, stride=2)),
])
def test_msssim_deep_inputs_vs_oracle(cuda, oracle, rng, bd, levels, window):
    from paper_2101_06354_b200 import synth

    h, w = 11 * 16 + 9, 11 * 16 + 37
    peak = (1 << bd) - 1
    base = synth.inv_f_noise(rng, h, w, float(peak))
    a = base.astype(np.uint16 if bd > 8 else np.uint8)
    b = np.clip(base + rng.normal(0, peak / 40, base.shape), 0, peak).round().astype(a.dtype)
    cfg = P.SsimConfig(bit_depth=bd, window=window)
    win = dict(shape=window.shape, k=window.k, stride=window.stride, sigma=window.sigma, bit_depth=bd)
    got = P.scale_scores(P.LumaPlane(a, bd), P.LumaPlane(b, bd), cfg, levels)
    want = oracle.scale_scores(a, b, levels, **win)
    tol = 1e-12 if window.shape == "rect" else 1e-5
    assert np.max(np.abs(np.array(got) - np.array(want))) < tol


def test_msssim_float_input_vs_oracle(cuda, oracle, rng):
    a = rng.uniform(0, 255, (100, 120))
    b = np.clip(a + rng.normal(0, 8, a.shape), 0, 255)
    for window, tol in ((P.WindowSpec.rectangular(5), 1e-9), (P.WindowSpec.gaussian(1.5), 1e-5)):
        cfg = P.SsimConfig(window=window)
        win = dict(shape=window.shape, k=window.k, sigma=window.sigma)
        got = P.msssim(P.LumaPlane(a), P.LumaPlane(b), cfg, P.MultiscaleSpec.product(3))
        assert abs(got - oracle.msssim(a, b, 3, **win)) < tol


def test_batch_api_odd_counts_misaligned_widths_and_color(cuda, oracle, rng):
    import torch

    n, h, w = 5, 41, 77  # odd n (last frame pair half empty), width not a multiple of 16
    a = rng.integers(0, 256, (n, h, w)).astype(np.uint8)
    b = np.clip(a.astype(int) + rng.integers(-30, 31, a.shape), 0, 255).astype(np.uint8)
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    got = P.ssim_batch(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), cfg).cpu().numpy()
    want = np.array([oracle.ssim_score(a[i], b[i], shape="gauss", k=11, sigma=1.5) for i in range(n)])
    assert np.max(np.abs(got - want)) < 1e-5
    # channel-wise color on device batches (4:2:0 planes at their own resolution)
    ys = [torch.from_numpy(a).cuda(), torch.from_numpy(a[:, ::2, ::2].copy()).cuda(), torch.from_numpy(a[:, 1::2, ::2].copy()).cuda()]
    ds = [torch.from_numpy(b).cuda(), torch.from_numpy(b[:, ::2, ::2].copy()).cuda(), torch.from_numpy(b[:, 1::2, ::2].copy()).cuda()]
    rc = P.SsimConfig(window=P.WindowSpec.rectangular(5))
    cw = P.color_batch(ys, ds, rc, alpha=-0.3, beta=-0.3).cpu().numpy()
    fx = P.color_batch(ys, ds, rc, weights=(0.8, 0.1, 0.1)).cpu().numpy()
    for i in range(n):
        sc = oracle.channel_scores([t[i].cpu().numpy() for t in ys], [t[i].cpu().numpy() for t in ds], shape="rect", k=5)
        assert abs(cw[i] - oracle.channelwise(sc, -0.3, -0.3)) < 1e-12
        assert abs(fx[i] - oracle.fixed_weight(sc, (0.8, 0.1, 0.1))) < 1e-12


def test_host_batch_scorer_matches_device_batch(cuda, rng):
    import torch

    n = 11
    a = rng.integers(0, 256, (n, 96, 130)).astype(np.uint8)
    b = np.clip(a.astype(int) + rng.integers(-20, 21, a.shape), 0, 255).astype(np.uint8)
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    spec = P.MultiscaleSpec.product(3)
    scorer = P.HostBatchScorer(cfg, spec, mode="both", chunk=4)
    ms, ss = scorer(torch.from_numpy(a).pin_memory(), torch.from_numpy(b).pin_memory())
    ms_dev, terms = P.msssim_batch(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), cfg, spec, with_ssim=True)
    assert np.array_equal(ms, ms_dev.cpu().numpy())
    assert np.array_equal(ss[:, 0], terms.score.cpu().numpy())
    assert scorer.h2d_bytes == 2 * a.nbytes
    # submitted one batch ahead (the bench's e2e loop): different batches in flight on the
    # shared double-buffered chunks still score exactly like the synchronous call
    batches = [(np.roll(a, i, axis=0), np.roll(b, i, axis=0)) for i in range(4)]
    pend, got = None, []
    for ra, rb in batches:
        nxt = scorer.submit(torch.from_numpy(ra).pin_memory(), torch.from_numpy(rb).pin_memory())
        if pend is not None:
            got.append(pend.result())
        pend = nxt
    got.append(pend.result())
    for i, (gms, gss) in enumerate(got):
        assert np.array_equal(gms, np.roll(ms, i)) and np.array_equal(gss, np.roll(ss, i, axis=0))


def test_sequence_scorer_multiscale_and_temporal_pooler(cuda, oracle, rng):
    frames = [(rng.integers(0, 256, (64, 80)).astype(np.uint8), rng.integers(0, 256, (64, 80)).astype(np.uint8))
              for _ in range(7)]
    cfg = P.SsimConfig(window=P.WindowSpec.rectangular(5), multiscale=P.MultiscaleSpec.product(3), temporal_pool="hm")
    res = P.score_sequence([f[0] for f in frames], [f[1] for f in frames], cfg, batch_frames=3)
    want = np.array([oracle.msssim(a, b, 3, shape="rect", k=5) for a, b in frames])
    assert np.max(np.abs(res.scores - want)) < 1e-12
    assert abs(res.pooled - P.pool_temporal(want, "hm")) < 1e-12
    assert all(r.am is None for r in res.records)


# --- SSIM-3D rolling volumes (src/spatiotemporal.py) ----------------------------

def test_ssim3d_against_golden(cuda, golden):
    fa = [golden[f"vol/ref{i}"] for i in range(7)]
    fb = [golden[f"vol/dist{i}"] for i in range(7)]
    got = P.ssim3d_series(fa, fb, 3, P.SsimConfig(window=P.WindowSpec.rectangular(7))).scores
    assert np.max(np.abs(got - golden["vol/series_k3"])) < 1e-12
    got = P.ssim3d_series(fa, fb, 1, P.SsimConfig(window=P.WindowSpec.rectangular(5, stride=2))).scores
    assert np.max(np.abs(got - golden["vol/series_k1"])) < 1e-12
    vol = P.RollingVolume(4)
    for a, b in zip(fa, fb):
        P.push_frame(vol, P.LumaPlane(a), P.LumaPlane(b))
    assert vol.depth == 4
    st = vol.local_statistics(P.WindowSpec.rectangular(6))
    assert np.array_equal(np.stack([st.mu1, st.mu2, st.var1, st.var2, st.cov]), golden["vol/stats_k4_w6"])
    q = P.ssim3d_map(vol, P.WindowSpec.rectangular(6)).q_map.values
    assert np.array_equal(q, golden["vol/q_k4_w6"])  # exact integer sums + reference fp64 epilogue
    sums = vol.temporal_sums()
    direct = vol.direct_sums()
    assert all(np.array_equal(x, y) for x, y in zip(sums, direct))
    ma = [golden[f"vol/msref{i}"] for i in range(4)]
    mb = [golden[f"vol/msdist{i}"] for i in range(4)]
    got = P.msssim3d(ma, mb, 2, P.MultiscaleSpec.product(3), P.SsimConfig(window=P.WindowSpec.rectangular(5))).scores
    assert np.max(np.abs(got - golden["vol/ms3d"])) < 1e-12


def test_ssim3d_sharded_with_halo_equals_unsharded(cuda, golden):
    fa = [golden[f"vol/ref{i}"] for i in range(7)]
    fb = [golden[f"vol/dist{i}"] for i in range(7)]
    cfg = P.SsimConfig(window=P.WindowSpec.rectangular(7))
    full = P.ssim3d_series(fa, fb, 3, cfg).scores
    for world in (2, 3):
        parts = [P.ssim3d_series_shard(fa, fb, 3, r, world, cfg).scores for r in range(world)]
        assert np.array_equal(np.concatenate(parts), full)


def test_ssim3d_float_refresh_against_golden(cuda, golden):
    fa = [golden[f"vol/ref{i}"].astype(np.float64) / 3.0 for i in range(7)]
    fb = [golden[f"vol/dist{i}"].astype(np.float64) / 3.0 for i in range(7)]
    vol = P.RollingVolume(3, refresh_interval=4)
    got = []
    for a, b in zip(fa, fb):
        vol.push(a, b)
        got.append(float(P.ssim3d_map(vol, P.WindowSpec.rectangular(5)).q_map.values.mean()))
    assert np.max(np.abs(np.array(got) - golden["vol/series_float_refresh4"])) < 1e-10


def test_ssim3d_kt1_equals_framewise_and_errors(cuda, rng):
    frames = [(rng.integers(0, 256, (40, 50)).astype(np.uint8), rng.integers(0, 256, (40, 50)).astype(np.uint8))
              for _ in range(3)]
    cfg = P.SsimConfig(window=P.WindowSpec.rectangular(7))
    s3 = P.ssim3d_series([a for a, _ in frames], [b for _, b in frames], 1, cfg).scores
    s2 = np.array([P.ssim_score(a, b, cfg) for a, b in frames])
    assert np.max(np.abs(s3 - s2)) < 1e-12
    vol = P.RollingVolume(2)
    with pytest.raises(ValidationError):
        vol.local_statistics(P.WindowSpec.rectangular(3))  # nothing buffered
    vol.push(*frames[0])
    from paper_2101_06354_b200.errors import GaussianNotSupported3D

    with pytest.raises(GaussianNotSupported3D):
        vol.local_statistics(P.WindowSpec.gaussian(1.5))
    with pytest.raises(ValidationError):
        vol.local_statistics(P.WindowSpec.rectangular(45))
    with pytest.raises(DimensionMismatch):
        vol.push(frames[0][0][:30], frames[0][1][:30])
    with pytest.raises(ValidationError):
        P.RollingVolume(0)


def test_ssim3d_cost_independent_of_kt(cuda, rng):
    """Acceptance criterion C4 (tests/test_acceptance.py:120-160): per-frame cost ~ independent of Kt."""
    import time

    import torch

    frames = [(rng.integers(0, 256, (256, 256)).astype(np.uint8), rng.integers(0, 256, (256, 256)).astype(np.uint8))
              for _ in range(24)]
    cfg = P.SsimConfig(window=P.WindowSpec.rectangular(8))

    def run(kt):
        vol = P.RollingVolume(kt)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for a, b in frames:
            vol.push(a, b)
            vol.terms(cfg.window, cfg)
        torch.cuda.synchronize()
        return time.perf_counter() - t0

    run(2)
    t2 = min(run(2) for _ in range(2))
    t10 = min(run(10) for _ in range(2))
    assert t10 / t2 < 1.5


def test_score_frame_pair_contract(cuda, oracle, rng, golden):
    a = rng.integers(0, 256, (60, 72)).astype(np.uint8)
    b = np.clip(a.astype(int) + rng.integers(-25, 26, a.shape), 0, 255).astype(np.uint8)
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    rec = P.score_frame_pair(P.LumaPlane(a), P.LumaPlane(b), cfg)
    want = oracle.ssim_terms(a, b, shape="gauss", k=11, sigma=1.5)
    assert abs(rec.score - want[0]) < 1e-5 and rec.am == rec.score
    assert abs(rec.l_mean - want[1]) < 1e-5 and abs(rec.cs_mean - want[2]) < 1e-5
    # non-mean spatial pooling pools the device map (and mean-luma map for lw)
    cfg_cov = P.SsimConfig(spatial_pool="cov")
    rec = P.score_frame_pair(a, b, cfg_cov)
    l_map, cs_map, q = oracle.ssim_maps(a, b)
    assert abs(rec.score - float(q.std() / q.mean())) < 1e-12
    mu1 = oracle.local_statistics(a, b, "rect", 11)[0]
    rec = P.score_frame_pair(a, b, P.SsimConfig(spatial_pool="lw:a=100,b=50"))
    wts = np.clip((mu1 - 100) / 50, 0, 1)
    assert abs(rec.score - float((wts * q).mean())) < 1e-12
    ms = P.score_frame_pair(a, b, P.SsimConfig(window=P.WindowSpec.rectangular(5), multiscale=P.MultiscaleSpec.product(3)))
    assert abs(ms.score - oracle.msssim(a, b, 3, shape="rect", k=5)) < 1e-12 and ms.am is None
    ref = P.ColorFrame(tuple(golden[f"color/ref{i}"] for i in range(3)), "ycbcr-bt709", "420")
    dist = P.ColorFrame(tuple(golden[f"color/dist{i}"] for i in range(3)), "ycbcr-bt709", "420")
    fx = P.score_frame_pair(ref, dist, P.SsimConfig(window=P.WindowSpec.gaussian(1.5),
                                                    color=P.ColorModelSpec("fixed", weights=(4 / 6, 1 / 6, 1 / 6))))
    assert abs(fx.score - float(golden["color/fixed"])) < 1e-5
    vol = P.RollingVolume(2)
    r3 = P.score_frame_pair(a, b, P.SsimConfig(window=P.WindowSpec.rectangular(7)), volume=vol)
    assert abs(r3.score - oracle.ssim_score(a, b, shape="rect", k=7)) < 1e-12
    with pytest.raises(ValidationError):
        P.score_frame_pair(a, b, P.SsimConfig(color=P.ColorModelSpec("qssim")))
    # resolution adaptation is on the device path now (tests/test_gpu_pool.py); frames
    # under 384 lines keep factor 1 under the 256-line rule
    if min(a.shape) < 384:
        scaled = P.score_frame_pair(a, b, P.SsimConfig(scaling=P.ScalePolicy.legacy256()))
        assert scaled.score == P.score_frame_pair(a, b, P.SsimConfig()).score


def test_score_files_y4m(cuda, oracle, tmp_path):
    from paper_2101_06354_b200 import ingest, synth

    vid = synth.VideoConfig3(frames=5, h=48, w=64)
    pairs = [vid.pair(t) for t in range(5)]
    ingest.write_y4m(tmp_path / "r.y4m", [r for r, _ in pairs], 64, 48)
    ingest.write_y4m(tmp_path / "d.y4m", [d for _, d in pairs], 64, 48)
    ref, dist = ingest.open_y4m(tmp_path / "r.y4m"), ingest.open_y4m(tmp_path / "d.y4m")
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    wts = (4 / 6, 1 / 6, 1 / 6)
    res = ingest.score_files(ref, dist, cfg, batch_frames=2, color_weights=wts)
    win = dict(shape="gauss", k=11, sigma=1.5)
    want = [oracle.fixed_weight(oracle.channel_scores(r, d, **win), wts) for r, d in pairs]
    assert np.max(np.abs(res.scores - np.array(want))) < 1e-5
    luma = ingest.score_files(ref, dist, cfg, batch_frames=3)
    assert np.max(np.abs(luma.scores - np.array([oracle.ssim_score(r[0], d[0], **win) for r, d in pairs]))) < 1e-5


def test_4k_config5_properties(cuda):
    """Config 5 at full size, through size-independent properties: unit score at identity,
    exact ref/dist symmetry, and batch invariance (a frame's scores do not depend on its
    batch neighbours) for Gaussian SSIM + 5-scale MS-SSIM on 3840x2160 u8."""
    import torch
    from paper_2101_06354_b200 import synth

    pairs = [synth.dct_pair(5, i, 2160, 3840) for i in range(2)]
    ref = torch.from_numpy(np.stack([pairs[0][0], pairs[1][0], pairs[0][0]])).to(cuda)
    dist = torch.from_numpy(np.stack([pairs[0][1], pairs[1][1], pairs[0][0]])).to(cuda)
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    spec = P.MultiscaleSpec.product(5)
    ms, terms = P.msssim_batch(ref, dist, cfg, spec, with_ssim=True)
    ms_sw, terms_sw = P.msssim_batch(dist, ref, cfg, spec, with_ssim=True)
    assert torch.equal(ms, ms_sw) and torch.equal(terms.score, terms_sw.score)  # exact symmetry
    assert abs(float(ms[2]) - 1.0) < 1e-6 and abs(float(terms.score[2]) - 1.0) < 1e-6  # identity
    alone, alone_t = P.msssim_batch(ref[1:2], dist[1:2], cfg, spec, with_ssim=True)
    assert float(alone[0]) == float(ms[1]) and float(alone_t.score[0]) == float(terms.score[1])
    assert 0.0 < float(ms[0]) < 1.0 and 0.0 < float(terms.score[0]) < 1.0


def _adversarial_pairs():
    h, w = 120, 520  # >= 490 columns: the wide (persistent) u8 kernel, fused level 1
    yy, xx = np.mgrid[0:h, 0:w]
    grad = ((xx * 255) // (w - 1)).astype(np.uint8)
    check = (((yy // 4 + xx // 4) % 2) * 255).astype(np.uint8)
    tex = np.random.default_rng(5).integers(0, 256, (h, w))
    return {
        "flat_equal": (np.full((h, w), 77, np.uint8), np.full((h, w), 77, np.uint8)),
        "flat_extremes": (np.zeros((h, w), np.uint8), np.full((h, w), 255, np.uint8)),
        "checker_inverted": (check, (255 - check).astype(np.uint8)),
        "gradient_plus_one": (grad, np.clip(grad.astype(int) + 1, 0, 255).astype(np.uint8)),
        "identical_texture": (check, check.copy()),
        "saturated_vs_texture": (np.full((h, w), 255, np.uint8), check),
        # large flat ref/dist offsets: Var(x - y) = E[b^2] - E[b]^2 would cancel without the
        # tile's difference shift d (sum / difference form of the score path); with opposite
        # offsets in the two halves of every tile d cannot follow both
        "offset_bright_vs_dark": ((tex // 4 + 180).astype(np.uint8), (tex // 4).astype(np.uint8)),
        "offset_opposite_halves": (np.where(xx < w // 2, tex // 2 + 60, tex // 2).astype(np.uint8),
                                   np.where(xx < w // 2, tex // 2, tex // 2 + 60).astype(np.uint8)),
    }


@pytest.mark.parametrize("name", sorted(_adversarial_pairs()))
def test_gaussian_adversarial_inputs_vs_oracle(cuda, oracle, name):
    """Flat windows (sigma ~ 0), extreme contrasts, exact identity and a near-flat gradient far
    from mid-gray through the fused Gaussian path (per-tile sample shift, C2 carried by the
    filter, sum / difference epilogue, fp32 tile sums): maps within 1e-4, scores within 1e-5 of
    the float64 oracle; MS-SSIM as well.  (With the fixed L/2 shift the gradient case was
    1.4e-4 off in cs and the shifted luminance form 3e-4 off in l.)"""
    a, b = _adversarial_pairs()[name]
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    win = dict(shape="gauss", k=11, sigma=1.5)
    got = P.ssim_map(a, b, cfg)
    want = oracle.ssim_maps(a, b, **win)
    for g, w_ in zip((got.l_map.values, got.cs_map.values, got.q_map.values), want):
        assert np.max(np.abs(g - w_)) < MAP_TOL
    terms = P.ssim_terms(a, b, cfg)
    assert max(abs(x - y) for x, y in zip(terms, oracle.ssim_terms(a, b, **win))) < SCORE_TOL
    assert abs(P.msssim(a, b, cfg, P.MultiscaleSpec.product(3)) - oracle.msssim(a, b, 3, **win)) < SCORE_TOL


@pytest.mark.parametrize("want_maps", [False, True])
@pytest.mark.parametrize("h,w", [(300, 520), (1080, 1920), (64, 700)])
def test_workspace_query_covers_every_launch(cuda, h, w, want_maps):
    """ssk_ssim_workspace_bytes must cover map launches too (they run on narrower strips,
    i.e. more partials, than score-only launches of the wide u8 kernel): a workspace of
    exactly the queried size works for both (the cached pool in engine would hide a short
    query in a long test session)."""
    import ctypes

    import torch
    from paper_2101_06354_b200 import _native as nat

    rng = np.random.default_rng(h + w)
    a = torch.from_numpy(rng.integers(0, 256, (2, h, w)).astype(np.uint8)).cuda()
    b = torch.from_numpy(rng.integers(0, 256, (2, h, w)).astype(np.uint8)).cuda()
    pair = engine.device_pair(a, b, 8, gauss=True)
    window = P.WindowSpec.gaussian(1.5)
    cfg = P.SsimConfig(window=window)
    lib = nat.lib()
    planes, win = pair.planes(), nat.make_window(window, cfg.c1, cfg.c2)
    size = lib.ssk_ssim_workspace_bytes(ctypes.byref(planes), ctypes.byref(win))
    ws = torch.empty(size, dtype=torch.uint8, device="cuda")
    want = nat.WANT_Q | nat.WANT_L | nat.WANT_CS
    sums = torch.empty((2, 3), dtype=torch.float64, device="cuda")
    maps = None
    if want_maps:
        gh, gw = engine.grid_shape(h, w, 11, 1)
        maps = torch.empty((2, 3, gh, gw), dtype=torch.float32, device="cuda")
        want |= nat.MAP_TERMS
    rc = lib.ssk_ssim(ctypes.byref(planes), ctypes.byref(win), want, sums.data_ptr(),
                      None if maps is None else maps.data_ptr(), ws.data_ptr(), ws.numel(),
                      nat.stream_handle(None))
    assert rc == 0, nat.lib().ssk_strerror(rc)


@pytest.mark.parametrize("bar", [20, 64, 150])
def test_gaussian_letterbox_bars_vs_oracle(cuda, oracle, bar):
    """Near-flat dark bars (0-2 noise) above 1/f content: the map launches shift every 8-row
    chunk by its own rows' level (a bar edge inside a tile no longer cancels in fp32; was up
    to 3e-4 off in cs with one shift per tile); scores (per-tile shift) within 1e-5."""
    from paper_2101_06354_b200 import synth

    rng = np.random.default_rng(bar)
    a = synth.inv_f_noise(rng, 300, 520, 255.0).astype(np.uint8)
    a[:bar] = rng.integers(0, 3, (bar, 520))
    b = np.clip(a.astype(int) + rng.integers(-1, 2, a.shape), 0, 255).astype(np.uint8)
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    win = dict(shape="gauss", k=11, sigma=1.5)
    got = P.ssim_map(a, b, cfg)
    for g, w_ in zip((got.l_map.values, got.cs_map.values, got.q_map.values), oracle.ssim_maps(a, b, **win)):
        assert np.max(np.abs(g - w_)) < MAP_TOL
    terms = P.ssim_terms(a, b, cfg)
    assert max(abs(x - y) for x, y in zip(terms, oracle.ssim_terms(a, b, **win))) < SCORE_TOL


@pytest.mark.parametrize("k,s", [(8, 4), (8, 2), (11, 1)])
def test_workspace_query_covers_q2_launches(cuda, oracle, k, s):
    """A Σq² launch (CoV / MD(2) pooling, rect windows) may take the per-window kernel, which
    makes more partials than the block kernel the score-only plan picks: a workspace of
    exactly the queried size must still work (1080p, rect 8 stride 4, cov)."""
    import ctypes

    import torch
    from paper_2101_06354_b200 import _native as nat

    rng = np.random.default_rng(k * 10 + s)
    h, w = 1080, 1920
    a_np = rng.integers(0, 256, (1, h, w)).astype(np.uint8)
    b_np = np.clip(a_np.astype(int) + rng.integers(-30, 31, a_np.shape), 0, 255).astype(np.uint8)
    a, b = torch.from_numpy(a_np).cuda(), torch.from_numpy(b_np).cuda()
    pair = engine.device_pair(a, b, 8, gauss=False)
    window = P.WindowSpec.rectangular(k, stride=s)
    cfg = P.SsimConfig(window=window)
    lib = nat.lib()
    planes, win = pair.planes(), nat.make_window(window, cfg.c1, cfg.c2)
    size = lib.ssk_ssim_workspace_bytes(ctypes.byref(planes), ctypes.byref(win))
    ws = torch.empty(size, dtype=torch.uint8, device="cuda")
    sums = torch.empty((1, 4), dtype=torch.float64, device="cuda")
    rc = lib.ssk_ssim(ctypes.byref(planes), ctypes.byref(win), nat.WANT_Q | nat.WANT_Q2, sums.data_ptr(),
                      None, ws.data_ptr(), ws.numel(), nat.stream_handle(None))
    assert rc == 0, nat.lib().ssk_strerror(rc)
    q = oracle.ssim_maps(a_np[0], b_np[0], shape="rect", k=k, stride=s)[2]
    got = sums.cpu().numpy()[0]
    assert abs(got[0] - q.sum()) < 1e-9 * q.size and abs(got[3] - (q * q).sum()) < 1e-9 * q.size


@pytest.mark.parametrize("sigma,k,stride,bd,kind", [
    (6.0, 37, 1, 8, "u8"), (6.0, 37, 3, 8, "u8"), (10.0, 61, 1, 10, "u16"), (5.5, 35, 2, 8, "f32"),
])
def test_wide_gaussian_windows_vs_oracle(cuda, oracle, sigma, k, stride, bd, kind):
    """Gaussian windows wider than 31 taps (the reference accepts any odd k >= 3,
    src/config.py:55-56): the generic fp64 kernel, maps and scores against the oracle,
    strided grids equal to dense[::s, ::s] exactly."""
    from paper_2101_06354_b200 import synth

    rng = np.random.default_rng(k * 7 + stride)
    peak = (1 << bd) - 1
    h, w = 150, 230
    a = synth.inv_f_noise(rng, h, w, float(peak))
    b = np.clip(a + rng.normal(0.0, peak / 40.0, a.shape), 0, peak)
    if kind == "f32":
        a, b = (a * 0.99 + 0.3).astype(np.float32), b.astype(np.float32)
    else:
        dt = np.uint8 if kind == "u8" else np.uint16
        a, b = a.astype(dt), np.round(b).astype(dt)
    window = P.WindowSpec.gaussian(sigma, k=k, stride=stride)
    cfg = P.SsimConfig(bit_depth=bd, window=window)
    ra, rb = P.LumaPlane(a, bd), P.LumaPlane(b, bd)
    maps = P.ssim_map(ra, rb, cfg)
    win = dict(shape="gauss", k=k, sigma=sigma, stride=stride, bit_depth=bd)
    wl, wcs, wq = oracle.ssim_maps(a, b, **win)
    assert maps.q_map.values.shape == wq.shape
    for got, want in ((maps.l_map.values, wl), (maps.cs_map.values, wcs), (maps.q_map.values, wq)):
        assert np.max(np.abs(got - want)) < 1e-6   # fp64 kernel, fp32 map store
    terms = P.ssim_terms(ra, rb, cfg)
    assert max(abs(x - y) for x, y in zip(terms, oracle.ssim_terms(a, b, **win))) < 1e-9
    st = P.local_statistics(ra, rb, window)
    want_st = oracle.local_statistics(a, b, "gauss", k, stride, sigma)
    assert np.max(np.abs(st.mu1 - want_st[0])) < 1e-3 * peak / 255
    assert np.max(np.abs(st.cov - want_st[4])) < 1e-2 * (peak / 255) ** 2
    if stride > 1:
        dense = P.ssim_map(ra, rb, P.SsimConfig(bit_depth=bd, window=P.WindowSpec.gaussian(sigma, k=k))).q_map.values
        assert np.array_equal(dense[::stride, ::stride], maps.q_map.values)


def test_wide_gaussian_msssim_vs_oracle(cuda, oracle):
    """MS-SSIM with a 37-tap window: every level on the generic kernel (no fused level 1)."""
    from paper_2101_06354_b200 import synth

    rng = np.random.default_rng(37)
    a = synth.inv_f_noise(rng, 160, 300, 255.0).astype(np.uint8)
    b = np.clip(a.astype(int) + rng.integers(-20, 21, a.shape), 0, 255).astype(np.uint8)
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(6.0))
    got = P.scale_scores(a, b, cfg, 2)
    want = oracle.scale_scores(a, b, 2, shape="gauss", k=37, sigma=6.0)
    assert np.max(np.abs(np.array(got) - np.array(want))) < 1e-9
    import torch

    ms = P.msssim_batch(torch.from_numpy(a[None]).cuda(), torch.from_numpy(b[None]).cuda(), cfg,
                        P.MultiscaleSpec.product(2))
    assert abs(float(ms[0]) - oracle.msssim(a, b, 2, shape="gauss", k=37, sigma=6.0)) < 1e-9


def _float_adversarial():
    h, w = 160, 520
    yy, xx = np.mgrid[0:h, 0:w]
    rng = np.random.default_rng(99)
    grad = (18.0 + 4.0 * xx / (w - 1)).astype(np.float32)            # near-flat, mu ~ 20
    from paper_2101_06354_b200 import synth

    content = synth.inv_f_noise(rng, h, w, 255.0).astype(np.float32)
    bars = content.copy()
    bars[:60] = rng.uniform(0.0, 2.0, (60, w)).astype(np.float32)    # dark letterbox bar
    bright = np.full((h, w), 236.0, np.float32) + rng.uniform(0, 0.5, (h, w)).astype(np.float32)
    return {
        "gradient_mu20": (grad, (grad + np.float32(0.37)).astype(np.float32)),
        "letterbox": (bars, np.clip(bars + rng.normal(0, 0.3, bars.shape), 0, 255).astype(np.float32)),
        "bright_flat": (bright, np.clip(bright + rng.normal(0, 0.2, bright.shape), 0, 255).astype(np.float32)),
    }


@pytest.mark.parametrize("name", sorted(_float_adversarial()))
def test_float_input_adversarial_vs_oracle(cuda, oracle, name):
    """float32 samples get the per-tile symmetric shift too (was a fixed L/2: a near-flat
    gradient at mu ~ 20 cancelled in fp32, 1.4e-4 off in cs): maps within 1e-4, scores
    and 3-scale MS-SSIM within 1e-5 of the float64 oracle."""
    a, b = _float_adversarial()[name]
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    win = dict(shape="gauss", k=11, sigma=1.5)
    got = P.ssim_map(a, b, cfg)
    for g, w_ in zip((got.l_map.values, got.cs_map.values, got.q_map.values), oracle.ssim_maps(a, b, **win)):
        assert np.max(np.abs(g - w_)) < MAP_TOL
    terms = P.ssim_terms(a, b, cfg)
    assert max(abs(x - y) for x, y in zip(terms, oracle.ssim_terms(a, b, **win))) < SCORE_TOL
    assert abs(P.msssim(a, b, cfg, P.MultiscaleSpec.product(3)) - oracle.msssim(a, b, 3, **win)) < SCORE_TOL


@pytest.mark.parametrize("bar", [0, 120])
def test_10bit_msssim_dark_letterbox_u32_level(cuda, oracle, bar):
    """10-bit 5-scale MS-SSIM: the coarsest level holds u32 sums of 256 samples (the per-tile
    shift now covers u32 levels); a dark near-flat letterbox bar above the content."""
    from paper_2101_06354_b200 import synth

    rng = np.random.default_rng(1000 + bar)
    h, w = 480, 704
    a = synth.inv_f_noise(rng, h, w, 1023.0)
    if bar:
        a[:bar] = rng.integers(0, 4, (bar, w))
    b = np.clip(a + rng.integers(-2, 3, a.shape), 0, 1023)
    a, b = a.astype(np.uint16), b.astype(np.uint16)
    cfg = P.SsimConfig(bit_depth=10, window=P.WindowSpec.gaussian(1.5))
    win = dict(shape="gauss", k=11, sigma=1.5, bit_depth=10)
    ra, rb = P.LumaPlane(a, 10), P.LumaPlane(b, 10)
    got = P.scale_scores(ra, rb, cfg, 5)
    want = oracle.scale_scores(a, b, 5, **win)
    assert np.max(np.abs(np.array(got) - np.array(want))) < SCORE_TOL


def test_score_only_bright_middle_row_over_dark(cuda, oracle):
    """score-only launches shift per tile from the tile's middle row; a bright band
    there over dark, near-flat content is the worst case for that choice (shift ~ L away
    from the dark windows' level).  Scores within 1e-5 of the oracle, and the score-only
    path agrees with the map path's mean."""
    rng = np.random.default_rng(5)
    h, w = 300, 520
    a = rng.integers(0, 3, (h, w)).astype(np.uint8)
    for r0 in (44, 140, 240):                      # near every segment's middle row
        a[r0:r0 + 16] = 250 + rng.integers(0, 5, (16, w))
    b = np.clip(a.astype(int) + rng.integers(-1, 2, a.shape), 0, 255).astype(np.uint8)
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    win = dict(shape="gauss", k=11, sigma=1.5)
    terms = P.ssim_terms(a, b, cfg)
    want = oracle.ssim_terms(a, b, **win)
    assert max(abs(x - y) for x, y in zip(terms, want)) < SCORE_TOL
    q = P.ssim_map(a, b, cfg).q_map.values
    assert abs(float(q.mean()) - terms[0]) < SCORE_TOL


@pytest.mark.parametrize("k,sigma,s,kind,h,w", [
    (11, 1.5, 2, "u8", 131, 517), (11, 1.5, 5, "u8", 300, 700), (11, 1.5, 3, "u16", 97, 260),
    (7, 1.0, 8, "u8", 120, 333), (31, 5.0, 4, "u8", 150, 600), (11, 1.5, 13, "u8", 90, 400),
    (3, 0.5, 2, "u16", 40, 300), (11, 1.5, 5, "u16", 1080, 1920),
])
def test_strided_gaussian_scores_vs_oracle(cuda, oracle, k, sigma, s, kind, h, w):
    """Strided Gaussian score launches run the anchor-only kernel (K1s): SSIM terms of an odd
    batch (a lone frame in the last packed pair) within 1e-5 of the float64 oracle, strides
    below, equal to and above k, 8- and 16-bit samples, strips and segments with ragged edges;
    MS-SSIM with a strided window at every level too."""
    import torch
    from paper_2101_06354_b200 import synth

    rng = np.random.default_rng(k * 1000 + s * 10 + h)
    bd = 8 if kind == "u8" else 10
    peak = (1 << bd) - 1
    dt = np.uint8 if kind == "u8" else np.uint16
    frames = []
    for _ in range(3):
        a = synth.inv_f_noise(rng, h, w, float(peak))
        b = np.clip(np.round(a + rng.normal(0, peak / 30.0, a.shape)), 0, peak)
        frames.append((a.astype(dt), b.astype(dt)))
    cfg = P.SsimConfig(bit_depth=bd, window=P.WindowSpec.gaussian(sigma, k=k, stride=s))
    ref = torch.from_numpy(np.stack([f[0] for f in frames])).to(cuda)
    dist = torch.from_numpy(np.stack([f[1] for f in frames])).to(cuda)
    t = P.ssim_terms_batch(ref, dist, cfg)
    got = np.stack([t.score.cpu().numpy(), t.l_mean.cpu().numpy(), t.cs_mean.cpu().numpy()], axis=1)
    win = dict(shape="gauss", k=k, sigma=sigma, stride=s, bit_depth=bd)
    for i, (a, b) in enumerate(frames):
        assert np.max(np.abs(got[i] - np.array(oracle.ssim_terms(a, b, **win)))) < SCORE_TOL, i
    if min(h, w) // 4 >= k:
        ms = P.msssim_batch(ref, dist, cfg, P.MultiscaleSpec.product(3)).cpu().numpy()
        for i, (a, b) in enumerate(frames):
            assert abs(ms[i] - oracle.msssim(a, b, 3, **win)) < SCORE_TOL, i
    # the map path (K1, anchor masking) agrees with the anchor-only scores
    q = P.ssim_map(P.LumaPlane(frames[0][0], bd), P.LumaPlane(frames[0][1], bd), cfg).q_map.values
    assert abs(float(q.mean()) - got[0, 0]) < SCORE_TOL


@pytest.mark.parametrize("name", ["gauss11", "gauss_s3", "gauss13_10b"])
def test_gaussian_map_api_is_fp64(cuda, golden, name):
    """ssim_map / local_statistics (the reference's map API) compute Gaussian maps with the
    fp64 kernel (SSK_MAP_F64): within 1e-12 of the reference's float64 maps, not just 1e-4."""
    cfg, bd, _ = CASES[name]
    ra, rb = planes(golden, name, bd)
    maps = P.ssim_map(ra, rb, cfg)
    for key, got in (("l", maps.l_map.values), ("cs", maps.cs_map.values), ("q", maps.q_map.values)):
        assert got.dtype == np.float64
        assert np.max(np.abs(got - golden[f"{name}/{key}"])) < 1e-12
    st = P.local_statistics(ra, rb, cfg.window, cfg.engine)
    want = golden[f"{name}/stats"]
    scale = float((1 << bd) - 1) ** 2
    for i, got in enumerate((st.mu1, st.mu2, st.var1, st.var2, st.cov)):
        assert np.max(np.abs(got - want[i])) < 1e-12 * scale


@pytest.mark.parametrize("bar", [20, 150])
def test_fp32_map_kernel_letterbox_vs_oracle(cuda, oracle, bar):
    """The fp32 K1 map launches (used inside batch pooling; per-chunk sample shift) on dark
    letterbox bars: maps within 1e-4 of the float64 oracle."""
    import torch
    from paper_2101_06354_b200 import _native as nat
    from paper_2101_06354_b200 import synth

    rng = np.random.default_rng(bar + 1)
    a = synth.inv_f_noise(rng, 300, 520, 255.0).astype(np.uint8)
    a[:bar] = rng.integers(0, 3, (bar, 520))
    b = np.clip(a.astype(int) + rng.integers(-1, 2, a.shape), 0, 255).astype(np.uint8)
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    pair = engine.device_pair(torch.from_numpy(a[None]).cuda(), torch.from_numpy(b[None]).cuda(), 8, gauss=True)
    _, maps = engine.ssim(pair, cfg.window, cfg.c1, cfg.c2, nat.WANT_Q | nat.MAP_TERMS)
    assert maps.dtype == torch.float32
    m = maps[0].double().cpu().numpy()
    wl, wcs, wq = oracle.ssim_maps(a, b, shape="gauss", k=11, sigma=1.5)
    for g, w_ in zip(m, (wl, wcs, wq)):
        assert np.max(np.abs(g - w_)) < MAP_TOL


def test_stats_and_term_maps_api_bit_exact(cuda, oracle, rng):
    """stats_from_sums / term_maps_from_stats run on the fp64 elementwise kernels in the
    reference's operation order: bit-identical to numpy's evaluation (oracle), including the
    variance clamp and broadcasting of a scalar sum."""
    from paper_2101_06354_b200 import moments, scoring

    shape = (37, 53)
    s1, s2 = rng.uniform(0, 255 * 121, shape), rng.uniform(0, 255 * 121, shape)
    q1 = s1 * s1 / 121 + rng.uniform(-5, 500, shape)  # some windows clamp at 0
    q2, p12 = s2 * s2 / 121 + rng.uniform(0, 500, shape), s1 * s2 / 121 + rng.uniform(-300, 300, shape)
    got = moments.stats_from_sums(s1, s2, q1, q2, p12, 121.0)
    want = oracle.moments_from_sums(s1, s2, q1, q2, p12, 121.0)
    for g, w_ in zip(got, want):
        assert np.array_equal(g, w_)
    st = P.LocalStatsMaps(mu1=want[0], mu2=want[1], var1=want[2], var2=want[3], cov=want[4], window_size=11,
                          stride=1, source_dims=(47, 63))
    maps = scoring.term_maps_from_stats(st, 6.5025, 58.5225)
    wl, wcs, wq = oracle.term_maps(*want, 6.5025, 58.5225)
    assert np.array_equal(maps.l_map.values, wl) and np.array_equal(maps.cs_map.values, wcs)
    assert np.array_equal(maps.q_map.values, wq)
    one = moments.stats_from_sums(np.float64(10.0), s2, q1, q2, p12, 121.0)[0]
    assert one.shape == shape and np.all(one == 10.0 / 121.0)


def test_c_host_program_end_to_end(cuda, oracle, tmp_path):
    """A C program using only the C ABI + the CUDA runtime (tests/c_abi/ssim_cli.c: library-built
    Gaussian taps from sigma, ssk_ssim + ssk_msssim) scores a pair like the oracle does."""
    import subprocess
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from test_native_abi import build_c_cli
    from paper_2101_06354_b200 import synth

    exe = build_c_cli(tmp_path)
    rng = np.random.default_rng(99)
    h, w = 300, 517
    a = synth.inv_f_noise(rng, h, w, 255.0).astype(np.uint8)
    b = np.clip(a.astype(int) + rng.integers(-15, 16, a.shape), 0, 255).astype(np.uint8)
    (tmp_path / "a.u8").write_bytes(a.tobytes())
    (tmp_path / "b.u8").write_bytes(b.tobytes())
    r = subprocess.run([str(exe), str(h), str(w), str(tmp_path / "a.u8"), str(tmp_path / "b.u8"), "1.5", "3"],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    f = r.stdout.split()
    win = dict(shape="gauss", k=11, sigma=1.5)
    assert max(abs(float(x) - y) for x, y in zip(f[1:4], oracle.ssim_terms(a, b, **win))) < SCORE_TOL
    assert abs(float(f[5]) - oracle.msssim(a, b, 3, **win)) < SCORE_TOL
