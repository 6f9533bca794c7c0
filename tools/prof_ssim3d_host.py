"""Host-side profile of ssim3d_series (where the per-frame time goes)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2101_06354_b200 as P
from paper_2101_06354_b200 import synth

pairs = [synth.dct_pair(2, i) for i in range(8)]
fr = [pairs[i % 8][0] for i in range(200)]
fd = [pairs[i % 8][1] for i in range(200)]
cfg = P.SsimConfig(window=P.WindowSpec.rectangular(8))
P.ssim3d_series(fr[:10], fd[:10], 3, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
P.ssim3d_series(fr, fd, 3, cfg)
print(f"{len(fr) / (time.perf_counter() - t0):.0f} frames/s")
pr = cProfile.Profile()
pr.enable()
P.ssim3d_series(fr, fd, 3, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
