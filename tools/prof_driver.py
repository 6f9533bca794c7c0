"""Short, deterministic driver for ncu captures (never used for bench numbers).

  --mode step : 3 full bench steps (64x 1080p SSIM + 5-scale MS-SSIM) -> launch list / shares
  --mode l0   : the level-0 fused Gaussian SSIM kernel over the 64-frame batch, 3 launches
  --mode box  : config-4 shape: rect 8 stride 4 on 10-bit 4K u16, 32 frames, 3 launches
  --mode stride : Gaussian 11/1.5 stride 5 scores (K1s) over the 64-frame 1080p batch, 3 launches
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="step", choices=["step", "l0", "box", "stride"])
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()

    import numpy as np
    import torch

    import paper_2101_06354_b200 as P
    from paper_2101_06354_b200 import _native, engine, synth

    dev = torch.device("cuda", 0)
    if args.mode == "box":
        pairs = [synth.config4_pair(i, 2160, 3840) for i in range(2)]
        ref = np.stack([pairs[i % 2][0] for i in range(32)])
        dist = np.stack([pairs[i % 2][1] for i in range(32)])
        cfg = P.SsimConfig(bit_depth=10, window=P.WindowSpec.rectangular(8, stride=4), engine="integral")
        r, d = torch.from_numpy(ref).to(dev), torch.from_numpy(dist).to(dev)
        for _ in range(args.reps):
            P.ssim_terms_batch(r, d, cfg)
        torch.cuda.synchronize()
        return
    pairs = [synth.dct_pair(2, i) for i in range(8)]
    ref = np.stack([pairs[i % 8][0] for i in range(64)])
    dist = np.stack([pairs[i % 8][1] for i in range(64)])
    r, d = torch.from_numpy(ref).to(dev), torch.from_numpy(dist).to(dev)
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    if args.mode == "step":
        for _ in range(args.reps):
            P.msssim_batch(r, d, cfg, P.MultiscaleSpec.product(5), with_ssim=True)
    elif args.mode == "stride":
        cs = P.SsimConfig(window=P.WindowSpec.gaussian(1.5, stride=5))
        for _ in range(args.reps):
            P.ssim_terms_batch(r, d, cs)
    else:
        pair = engine.device_pair(r, d, 8, gauss=True)
        for _ in range(args.reps):
            engine.ssim(pair, cfg.window, cfg.c1, cfg.c2, _native.WANT_Q | _native.WANT_L | _native.WANT_CS)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
