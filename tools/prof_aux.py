"""Driver for ncu captures of the auxiliary kernels of the hot path: the levels 2-4
pyramid pass and the MS-SSIM finalize (one bench step), and the SSIM-3D rolling
volume update + box kernel over a short 1080p sequence."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import paper_2101_06354_b200 as P
from paper_2101_06354_b200 import synth

pairs = [synth.dct_pair(2, i) for i in range(8)]
ref = torch.from_numpy(np.stack([pairs[i % 8][0] for i in range(64)])).cuda()
dist = torch.from_numpy(np.stack([pairs[i % 8][1] for i in range(64)])).cuda()
cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
for _ in range(2):
    P.msssim_batch(ref, dist, cfg, P.MultiscaleSpec.product(5), with_ssim=True)
frames_r = [pairs[i % 8][0] for i in range(6)]
frames_d = [pairs[i % 8][1] for i in range(6)]
P.ssim3d_series(frames_r, frames_d, 3, P.SsimConfig(window=P.WindowSpec.rectangular(8)))
torch.cuda.synchronize()
