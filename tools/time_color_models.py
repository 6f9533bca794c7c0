"""Per-pair time of the colorimetric models at 1080p RGB u8 (rect 11)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2101_06354_b200 as P
from paper_2101_06354_b200 import synth

rng = np.random.default_rng(3)
rgb_r = tuple(synth.inv_f_noise(rng, 1080, 1920, 255.0).astype(np.uint8) for _ in range(3))
rgb_d = tuple(np.clip(c.astype(np.int16) + rng.integers(-8, 9, c.shape), 0, 255).astype(np.uint8) for c in rgb_r)
fr, fd = P.ColorFrame(rgb_r), P.ColorFrame(rgb_d)
for name, fn in (("qssim", lambda: P.qssim(fr, fd)), ("cmssim", lambda: P.cmssim(fr, fd)),
                 ("hssim", lambda: P.hssim(fr, fd))):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        v = fn()
    print(f"{name}: {(time.perf_counter() - t0) / 5 * 1e3:.2f} ms per pair, score {v!r}")
