"""Per-frame cost of SSIM-3D (rolling temporal sums + box window) on a 1080p u8 stream."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2101_06354_b200 as P
from paper_2101_06354_b200 import synth

pairs = [synth.dct_pair(2, i) for i in range(8)]
fr = [pairs[i % 8][0] for i in range(40)]
fd = [pairs[i % 8][1] for i in range(40)]
cfg = P.SsimConfig(window=P.WindowSpec.rectangular(8))
P.ssim3d_series(fr[:5], fd[:5], 3, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
s = P.ssim3d_series(fr, fd, 3, cfg).scores
dt = time.perf_counter() - t0
print(f"ssim3d kt=3 rect8 1080p: {len(fr) / dt:.0f} frames/s end to end (numpy frames in), mean {s.mean():.6f}")
