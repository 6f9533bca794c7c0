"""cProfile of the SequenceScorer host path (config-3 shape) to find host-side bottlenecks."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2101_06354_b200 as P  # noqa: E402
from paper_2101_06354_b200 import synth  # noqa: E402

vid = synth.VideoConfig3(frames=160)
pairs = [vid.pair(t) for t in range(160)]
cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
sc = P.SequenceScorer(cfg, batch_frames=16, color_weights=(4 / 6, 1 / 6, 1 / 6))
sc.score([r for r, _ in pairs[:32]], [d for _, d in pairs[:32]])
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
res = sc.score([r for r, _ in pairs], [d for _, d in pairs])
torch.cuda.synchronize()
pr.disable()
print("frames/s", 160 / (time.perf_counter() - t0))
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
