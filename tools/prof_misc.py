"""Small driver for ncu captures of the secondary kernels (enhanced preset, colorimetric, pooling)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import paper_2101_06354_b200 as P
from paper_2101_06354_b200 import synth

pool = [synth.dct_pair(2, i, 1080, 1920) for i in range(4)]
ref = torch.from_numpy(np.stack([pool[i % 4][0] for i in range(64)])).cuda()
dist = torch.from_numpy(np.stack([pool[i % 4][1] for i in range(64)])).cuda()
P.score_batch(ref, dist, P.expand_preset("enhanced").config)            # box_down_vec + box_int(Q2) + moments
rng = np.random.default_rng(3)
rgb = tuple(synth.inv_f_noise(rng, 1080, 1920, 255.0).astype(np.uint8) for _ in range(3))
rgb2 = tuple(np.clip(c.astype(np.int16) + 5, 0, 255).astype(np.uint8) for c in rgb)
P.qssim(P.ColorFrame(rgb), P.ColorFrame(rgb2))                          # color_convert + qssim
P.cmssim(P.ColorFrame(rgb), P.ColorFrame(rgb2))                         # opponent + smooth + delta_e
q = 1.0 - 0.05 * torch.rand((64, 1070, 1910), dtype=torch.float32, device="cuda") ** 3  # SSIM-like: crowded near 1
P.pool_maps(q, "fns")                                                    # radix select
P.pool_maps(q, "cov")                                                    # two-pass sums
torch.cuda.synchronize()
