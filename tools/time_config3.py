"""Config 3 end to end (300 1080p YUV420 frames, per-plane Gaussian SSIM, weights (4,1,1)/6,
temporal mean) through SequenceScorer from host numpy frames; repeated to show variance."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2101_06354_b200 as P
from paper_2101_06354_b200 import synth

cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
nfr = 300
vid = synth.VideoConfig3(frames=nfr)
pairs = [vid.pair(t) for t in range(nfr)]
scorer = P.SequenceScorer(cfg, batch_frames=16, color_weights=(4 / 6, 1 / 6, 1 / 6))
scorer.score([r for r, _ in pairs[:32]], [d for _, d in pairs[:32]])
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = scorer.score([r for r, _ in pairs], [d for _, d in pairs])
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"config3 rep {rep}: {nfr / dt:.0f} frames/s end to end, pooled {res.pooled:.6f}")
