"""Throughput of the other BASELINE.json configurations (not the driver's bench line).

  config1: 512x512 u8 Gaussian SSIM, one pair per call (latency of the per-pair API)
  config3: 1080p YUV420 video, per-plane Gaussian SSIM, fixed weights (4,1,1)/6, temporal mean,
           through SequenceScorer (numpy frames -> pinned ring -> H2D -> kernels)
  config4: 4K 10-bit u16 rect 8 stride 4 (integral engine semantics), device-resident batches
  config5: 4K u8 Gaussian SSIM + 5-scale MS-SSIM per pair, device-resident batches

Seeded pools of distinct pairs are cycled to fill the batches (generation of
4K 1/f-noise pairs is CPU-heavy); the pool size is printed.  Prints one JSON
object per configuration.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def _hbm_peak() -> float:
    """Measured HBM copy bandwidth of this pool (MEASURED_PEAKS.json, driver-written), GB/s."""
    p = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6552.3  # the value measured on this pool in round 1


HBM_PEAK = _hbm_peak()


def timed(fn, reps: int) -> float:
    import torch

    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def main() -> None:
    import numpy as np
    import torch

    import bench
    import paper_2101_06354_b200 as P
    from paper_2101_06354_b200 import synth

    dev = torch.device("cuda", 0)
    out = {}

    # config 1: per-pair API latency (host arrays in, score out)
    a, b = synth.config1_pair()
    cfg = P.SsimConfig(window=P.WindowSpec.gaussian(1.5))
    P.ssim_score(a, b, cfg)
    t0 = time.perf_counter()
    for _ in range(50):
        s = P.ssim_score(a, b, cfg)
    dt = (time.perf_counter() - t0) / 50
    out["config1"] = {"score": s, "ms_per_call": dt * 1e3, "path": "ssim_score(host numpy, 512x512 u8)"}

    # config 4: 4K 10-bit box windows, HBM-bound
    pool = [synth.config4_pair(i) for i in range(4)]
    n = 32
    ref = torch.from_numpy(np.stack([pool[i % 4][0] for i in range(n)])).to(dev)
    dist = torch.from_numpy(np.stack([pool[i % 4][1] for i in range(n)])).to(dev)
    cfg4 = P.SsimConfig(bit_depth=10, window=P.WindowSpec.rectangular(8, stride=4), engine="integral")
    sec = timed(lambda: P.ssim_terms_batch(ref, dist, cfg4), 20)
    bytes_per_pair = 2 * 2160 * 3840 * 2
    out["config4"] = {"pairs_per_s": n / sec, "hbm_GBps": n * bytes_per_pair / sec / 1e9,
                      "hbm_peak_GBps": HBM_PEAK, "hbm_frac": n * bytes_per_pair / sec / 1e9 / HBM_PEAK,
                      "batch": n, "pool": 4}
    del ref, dist

    # config 5: 4K u8 SSIM + MS-SSIM
    pool = [synth.dct_pair(5, i, 2160, 3840) for i in range(8)]
    n = 32
    ref = torch.from_numpy(np.stack([pool[i % 8][0] for i in range(n)])).to(dev)
    dist = torch.from_numpy(np.stack([pool[i % 8][1] for i in range(n)])).to(dev)
    spec = P.MultiscaleSpec.product(5)
    sec = timed(lambda: P.msssim_batch(ref, dist, cfg, spec, with_ssim=True), 10)
    flops = n * bench.msssim_flops(2160, 3840)
    out["config5"] = {"pairs_per_s": n / sec, "TFLOPs": flops / sec / 1e12, "batch": n, "pool": 8,
                      "note": "4800 pairs would take %.3f s on one GPU" % (4800 / (n / sec))}
    del ref, dist
    # the whole 4800-pair sweep resident in HBM (2 x 39.8 GB of 4K u8 frames), scored in
    # 300-frame launches: per-frame SSIM + MS-SSIM scores only leave the device at the end
    if "--no-sweep" not in sys.argv:
        total, chunk = 4800, 300
        big_r = torch.empty((total, 2160, 3840), dtype=torch.uint8, device=dev)
        big_d = torch.empty_like(big_r)
        pr = torch.from_numpy(np.stack([p[0] for p in pool])).to(dev)
        pd = torch.from_numpy(np.stack([p[1] for p in pool])).to(dev)
        for i in range(0, total, len(pool)):
            big_r[i:i + len(pool)].copy_(pr)
            big_d[i:i + len(pool)].copy_(pd)
        del pr, pd

        def sweep():
            outs = [P.msssim_batch(big_r[i:i + chunk], big_d[i:i + chunk], cfg, spec, with_ssim=True)
                    for i in range(0, total, chunk)]
            return torch.cat([o[0] for o in outs]), torch.cat([o[1].score for o in outs])

        sec = timed(sweep, 2)
        ms_scores, ss_scores = sweep()
        out["config5_resident_sweep"] = {
            "pairs": total, "seconds": sec, "pairs_per_s": total / sec, "hbm_resident_GB": 2 * big_r.numel() / 1e9,
            "msssim_mean": float(ms_scores.mean()), "ssim_mean": float(ss_scores.mean()), "chunk": chunk}
        del big_r, big_d
        torch.cuda.empty_cache()

    # enhanced preset (rect 11 stride 5, integral engine, dh:3 box downsampling, CoV pooling) at 1080p
    pool = [synth.dct_pair(2, i, 1080, 1920) for i in range(8)]
    n = 64
    ref = torch.from_numpy(np.stack([pool[i % 8][0] for i in range(n)])).to(dev)
    dist = torch.from_numpy(np.stack([pool[i % 8][1] for i in range(n)])).to(dev)
    enh = P.expand_preset("enhanced").config
    l0 = P.engine.launch_count()
    P.score_batch(ref, dist, enh)
    launches = P.engine.launch_count() - l0
    sec = timed(lambda: P.score_batch(ref, dist, enh), 50)
    out["enhanced"] = {"pairs_per_s": n / sec, "ms_per_batch": sec * 1e3, "batch": n, "pool": 8,
                       "hbm_GBps_input": n * 2 * 1080 * 1920 / sec / 1e9, "launches_per_batch": launches,
                       "path": "score_batch(enhanced preset): box downsample x4 -> rect11/s5 maps -> device CoV"}
    del ref, dist

    # colorimetric models: per-pair API at 1080p RGB (host frames in, score out)
    rng = np.random.default_rng(77)
    rgb_r = tuple(synth.inv_f_noise(rng, 1080, 1920, 255.0).astype(np.uint8) for _ in range(3))
    rgb_d = tuple(np.clip(c.astype(np.int16) + rng.integers(-8, 9, c.shape), 0, 255).astype(np.uint8) for c in rgb_r)
    fr, fd = P.ColorFrame(rgb_r), P.ColorFrame(rgb_d)
    for name, fn in (("qssim", lambda: P.qssim(fr, fd)), ("cmssim", lambda: P.cmssim(fr, fd)),
                     ("hssim", lambda: P.hssim(fr, fd))):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            v = fn()
        dt = (time.perf_counter() - t0) / 5
        out[name] = {"ms_per_pair": dt * 1e3, "score": v, "path": f"{name}(ColorFrame 1080p RGB u8), rect 11"}

    # config 3: YUV420 video through the frame-stream API (host frames -> pinned ring -> GPU)
    nfr = 300
    vid = synth.VideoConfig3(frames=nfr)
    pairs = [vid.pair(t) for t in range(nfr)]
    scorer = P.SequenceScorer(cfg, batch_frames=16, color_weights=(4 / 6, 1 / 6, 1 / 6))
    scorer.score([r for r, _ in pairs[:32]], [d for _, d in pairs[:32]])  # warm both pinned slots
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = scorer.score([r for r, _ in pairs], [d for _, d in pairs])
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    out["config3"] = {"frames_per_s_e2e": nfr / dt, "pooled": res.pooled, "frames": nfr,
                      "h2d_bytes": res.h2d_bytes, "path": "SequenceScorer(color_weights=(4,1,1)/6), host numpy frames"}
    # the same video as Y4M files: memory-mapped, page-locked in place, planes DMA'd with no host copy
    import tempfile

    from paper_2101_06354_b200 import ingest

    with tempfile.TemporaryDirectory() as td:
        ingest.write_y4m(f"{td}/r.y4m", [r for r, _ in pairs], 1920, 1080)
        ingest.write_y4m(f"{td}/d.y4m", [d for _, d in pairs], 1920, 1080)
        rs, ds = ingest.open_y4m(f"{td}/r.y4m"), ingest.open_y4m(f"{td}/d.y4m")
        pinned = rs.pin() and ds.pin()
        w = (4 / 6, 1 / 6, 1 / 6)
        ingest.score_files(rs, ds, cfg, 16, w)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res2 = ingest.score_files(rs, ds, cfg, 16, w)
        torch.cuda.synchronize()
        dt2 = time.perf_counter() - t0
        out["config3_files"] = {"frames_per_s_e2e": nfr / dt2, "pooled": res2.pooled, "frames": nfr,
                                "pinned_mapping": pinned, "h2d_GBps": res2.h2d_bytes / dt2 / 1e9,
                                "path": "score_files(open_y4m x2): mmap -> cudaHostRegister -> DMA per plane"}
        rs.close()
        ds.close()
    for k, v in out.items():
        print(json.dumps({"config": k, **v}), flush=True)


if __name__ == "__main__":
    main()
