"""Small cases for compute-sanitizer (racecheck / synccheck / memcheck / initcheck).

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]

Each case launches the kernels named beside it on inputs that exercise their hand-rolled
synchronisation (named-barrier rings, cp.async / cp.async.bulk + mbarrier rings,
multi-tile persistent CTAs) at sizes small enough for the sanitizers' slowdown.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import paper_2101_06354_b200 as P
from paper_2101_06354_b200 import synth


def _u8(rng, n, h, w):
    a = rng.integers(0, 256, (n, h, w)).astype(np.uint8)
    b = np.clip(a.astype(int) + rng.integers(-30, 31, a.shape), 0, 255).astype(np.uint8)
    return torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()


def persist_k1(rng):
    """gauss_ws_persist_kernel: 41 wide u8 frames -> 252 tiles, CTAs walk several tiles;
    with the fused level-1 stores (MS-SSIM) and without."""
    a, b = _u8(rng, 41, 512, 600)
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    P.ssim_terms_batch(a, b, cfg)
    P.msssim_batch(a[:9], b[:9], cfg, P.MultiscaleSpec.product(3))


def levels(rng):
    """gauss_levels_kernel (coarse u16 / u32 levels, wide + classic strips) and pyramid_kernel."""
    a, b = _u8(rng, 4, 1080, 1920)
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    P.msssim_batch(a, b, cfg, P.MultiscaleSpec.product(5))
    x = torch.from_numpy(rng.integers(0, 1024, (2, 480, 704)).astype(np.uint16)).cuda()
    y = torch.clamp(x + 3, max=1023)
    P.msssim_batch(x, y, P.SsimConfig(bit_depth=10, window=P.WindowSpec.gaussian(1.5)), P.MultiscaleSpec.product(5))


def maps(rng):
    """Classic K1 map launches (per-chunk shift) and the 5-moment statistics variant."""
    a, b = _u8(rng, 1, 300, 520)
    an, bn = a[0].cpu().numpy(), b[0].cpu().numpy()
    P.ssim_map(an, bn, P.SsimConfig(window=P.WindowSpec.gaussian(1.5)))
    P.local_statistics(an, bn, P.WindowSpec.gaussian(1.5))


def box(rng):
    """box_block kernel (cp.async.bulk + mbarrier ring) on a config-4 crop, box_int (stride
    not dividing k, q^2 sums) and the integral tables."""
    a, b = synth.config4_pair(0, 512, 1024)
    ta = torch.from_numpy(np.stack([a, b])).cuda()
    tb = torch.from_numpy(np.stack([b, a])).cuda()
    P.ssim_terms_batch(ta, tb, P.SsimConfig(bit_depth=10, window=P.WindowSpec.rectangular(8, stride=4),
                                            engine="integral"))
    P.score_frame_pair(P.LumaPlane(a, 10), P.LumaPlane(b, 10),
                       P.SsimConfig(bit_depth=10, window=P.WindowSpec.rectangular(11, stride=5), spatial_pool="cov"))
    P.build_integral_set(P.LumaPlane(a[:64, :96], 10), P.LumaPlane(b[:64, :96], 10))


def generic(rng):
    """gauss_generic_kernel (k > 31, fp64)."""
    a, b = _u8(rng, 2, 150, 230)
    P.ssim_terms_batch(a, b, P.SsimConfig(window=P.WindowSpec.gaussian(6.0)))
    an, bn = a[0].cpu().numpy(), b[0].cpu().numpy()
    P.ssim_map(an, bn, P.SsimConfig(window=P.WindowSpec.gaussian(6.0, stride=3)))


def pooling(rng):
    """select_hist / select_pick (radix select: fns, median) and the CoV sums."""
    q = 1.0 - 0.05 * torch.rand((3, 200, 300), dtype=torch.float32, device="cuda") ** 3
    for m in ("fns", "median", "cov"):
        P.pool_maps(q, m)


CASES = {f.__name__: f for f in (persist_k1, levels, maps, box, generic, pooling)}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    rng = np.random.default_rng(11)
    for n in names:
        CASES[n](rng)
        torch.cuda.synchronize()
        print("case", n, "ok", flush=True)
