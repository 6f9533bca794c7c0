"""Run the enhanced preset on a 64 x 1080p device batch (for ncu launch lists)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import paper_2101_06354_b200 as P
from paper_2101_06354_b200 import synth

pool = [synth.dct_pair(2, i, 1080, 1920) for i in range(8)]
ref = torch.from_numpy(np.stack([pool[i % 8][0] for i in range(64)])).cuda()
dist = torch.from_numpy(np.stack([pool[i % 8][1] for i in range(64)])).cuda()
cfg = P.expand_preset("enhanced").config
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    rec = P.score_batch(ref, dist, cfg)
torch.cuda.synchronize()
print(float(rec.score.mean()))
