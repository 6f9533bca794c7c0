"""Time Gaussian SSIM score launches on small / odd geometries (CUDA events, warm).
usage: python tools/time_small.py  (env switches such as SSK_GAUSS_WS apply)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2101_06354_b200 as P

rng = np.random.default_rng(3)
for n, h, w in ((256, 288, 352), (256, 240, 320), (64, 480, 480), (64, 540, 960), (16, 2160, 3840)):
    a = rng.integers(0, 256, (n, h, w)).astype(np.uint8)
    b = np.clip(a.astype(int) + rng.integers(-20, 21, a.shape), 0, 255).astype(np.uint8)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    for _ in range(3):
        P.ssim_terms_batch(ta, tb, cfg)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        P.ssim_terms_batch(ta, tb, cfg)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{n:4d} x {h}x{w}: {ms:.4f} ms per batch, {n / ms * 1e3 / 1e3:.1f} k pairs/s, {n * h * w / ms / 1e6:.1f} Gpx/s")
