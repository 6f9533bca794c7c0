"""Score error of the Gaussian path vs the float64 oracle for flat-ish content with opposite
ref/dist offsets in the two halves of every tile (the case the tile's difference shift d cannot follow)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

import paper_2101_06354_b200 as P
from oracle import ssim_oracle as O

h, w = 120, 520
yy, xx = np.mgrid[0:h, 0:w]
rng = np.random.default_rng(5)
cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
for amp, noise in ((60, 128), (120, 64), (200, 8), (200, 0), (250, 0)):
    tex = rng.integers(0, noise + 1, (h, w))
    a = np.where(xx < w // 2, tex + amp, tex).astype(np.uint8)
    b = np.where(xx < w // 2, tex, tex + amp).astype(np.uint8)
    got = P.ssim_terms(a, b, cfg)
    want = O.ssim_terms(a, b, shape="gauss", k=11, sigma=1.5)
    print(f"offset +-{amp}, texture 0..{noise}: |d score| {abs(got[0] - want[0]):.2e}  |d l| {abs(got[1] - want[1]):.2e}  "
          f"|d cs| {abs(got[2] - want[2]):.2e}")
