"""Letterbox check: dark bars (0..2 noise) above textured content, Gaussian maps vs the oracle."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2101_06354_b200 as P
from oracle import ssim_oracle as O
from paper_2101_06354_b200 import synth

rng = np.random.default_rng(5)
h, w = 300, 520
for bar in (20, 64, 100, 150):
    a = synth.inv_f_noise(rng, h, w, 255.0).astype(np.uint8)
    a[:bar] = rng.integers(0, 3, (bar, w))
    b = np.clip(a.astype(int) + rng.integers(-1, 2, a.shape), 0, 255).astype(np.uint8)
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    got = P.ssim_map(a, b, cfg)
    want = O.ssim_maps(a, b, shape="gauss", k=11, sigma=1.5)
    errs = [float(np.max(np.abs(g - w_))) for g, w_ in zip((got.l_map.values, got.cs_map.values, got.q_map.values), want)]
    t = P.ssim_terms(a, b, cfg)
    te = max(abs(x - y) for x, y in zip(t, O.ssim_terms(a, b, shape="gauss", k=11, sigma=1.5)))
    print(f"bar {bar}: map errs l/cs/q {errs[0]:.2e} {errs[1]:.2e} {errs[2]:.2e}  score err {te:.2e}")
