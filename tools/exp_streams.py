"""Experiment: one 64-pair MS-SSIM batch vs the same batch as 2 or 4 sub-batches on
separate streams (kernel tails of one sub-batch filled by the next one's CTAs)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2101_06354_b200 as P
from paper_2101_06354_b200 import synth

dev = torch.device("cuda", 0)
pairs = [synth.dct_pair(2, i) for i in range(8)]
ref = torch.from_numpy(np.stack([pairs[i % 8][0] for i in range(64)])).to(dev)
dist = torch.from_numpy(np.stack([pairs[i % 8][1] for i in range(64)])).to(dev)
cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
spec = P.MultiscaleSpec.product(5)
want = P.msssim_batch(ref, dist, cfg, spec, with_ssim=True)[0]
main = torch.cuda.current_stream()
for nsplit in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(nsplit)]
    b = 64 // nsplit

    def step():
        outs = []
        ev = torch.cuda.Event()
        ev.record(main)
        for i, s in enumerate(streams):
            s.wait_event(ev)
            outs.append(P.msssim_batch(ref[i * b:(i + 1) * b], dist[i * b:(i + 1) * b], cfg, spec, with_ssim=True,
                                       stream=s)[0])
        for s in streams:
            main.wait_stream(s)
        return outs

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(30):
        outs = step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 30
    same = torch.equal(torch.cat(outs), want)
    print(f"split {nsplit}: {ms:.4f} ms/step  {64 / ms * 1e3:.0f} pairs/s  identical={same}")
