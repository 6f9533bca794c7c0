"""Gaussian stride as a speed path: 1080p Gaussian 11/1.5 SSIM scores at s = 1, 2, 3, 4, 5, 8.

One JSON line per stride: pairs/s over a 64-frame config-2 batch (device-resident, CUDA
events around 20 launches after warm-up), the kernel's algorithmic FP32 rate (SURVEY.md 8(d)
count at that stride) against the in-run FFMA peak, and its HBM rate (2 H W bytes per pair)
against MEASURED_PEAKS.json.

    python tools/bench_stride.py
"""
import json
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

import numpy as np
import torch

import bench
import paper_2101_06354_b200 as P
from paper_2101_06354_b200 import _native


def main():
    lib = _native.load_library()
    ref_np, dist_np = bench.generate(range(64), 8)
    ref, dist = torch.from_numpy(ref_np).cuda(), torch.from_numpy(dist_np).cuda()
    peak = bench.ctypes_probe(lib, 1.0)
    try:
        hbm = json.loads((REPO / "MEASURED_PEAKS.json").read_text())
        hbm_peak = float(hbm["hbm_gbs"])
    except (OSError, ValueError):
        hbm_peak = 6462.7
    base = None
    for s in (1, 2, 3, 4, 5, 8):
        cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5, stride=s))
        for _ in range(3):
            P.ssim_terms_batch(ref, dist, cfg)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for _ in range(reps):
            t = P.ssim_terms_batch(ref, dist, cfg)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        rate = 64 / (ms * 1e-3)
        base = base or rate
        flops = 64 * bench.ssim_flops(1080, 1920, 11, s)
        print(json.dumps({"stride": s, "pairs_per_s": rate, "speedup_vs_s1": rate / base, "ms_per_batch": ms,
                          "fp32_tflops": flops / (ms * 1e-3) / 1e12, "fp32_frac": flops / (ms * 1e-3) / 1e12 / peak,
                          "hbm_gbps": 64 * 2 * 1080 * 1920 / (ms * 1e-3) / 1e9,
                          "hbm_frac": 64 * 2 * 1080 * 1920 / (ms * 1e-3) / 1e9 / hbm_peak,
                          "score_mean": float(t.score.mean())}), flush=True)


if __name__ == "__main__":
    main()
