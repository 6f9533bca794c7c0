"""Experiment: one 64-pair MS-SSIM step as 1, 2 or 4 sub-batches on side streams
(engine.msssim_levels(split=...)); run under SSK_GAUSS_PERSIST=0/1 to compare."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2101_06354_b200 as P
from paper_2101_06354_b200 import engine, synth

dev = torch.device("cuda", 0)
pairs = [synth.dct_pair(2, i) for i in range(8)]
ref = torch.from_numpy(np.stack([pairs[i % 8][0] for i in range(64)])).to(dev)
dist = torch.from_numpy(np.stack([pairs[i % 8][1] for i in range(64)])).to(dev)
cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
spec = P.MultiscaleSpec.product(5)
pair = engine.device_pair(ref, dist, 8, gauss=True)
want = None
for split in (1, 2, 3, 4):
    def step():
        return engine.msssim_levels(pair, cfg.window, cfg.c1, cfg.c2, 5, with_ssim=True, spec=spec, split=split)[1]

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(30):
        out = step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 30
    want = out if want is None else want
    print(f"split {split}: {ms:.4f} ms/step  {64 / ms * 1e3:.0f} pairs/s  identical={torch.equal(out, want)}")
