"""Golden vectors for the file pipeline: run_score over Y4M / raw / PNM inputs and the
report writer, produced by running the REFERENCE (ssimkit) itself.

    PYTHONPATH=/root/reference/pkg/src python -B tests/golden/make_golden_media.py

Writes tests/golden/golden_media_v1.npz: the frames (so the tests can rewrite the
same files), run_score records/summary values per spec, and write_report bytes.
"""

from __future__ import annotations

import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

from ssimkit.config import ColorModelSpec, MultiscaleSpec, SsimConfig, WindowSpec  # noqa: E402  (the reference)
from ssimkit.frames import ColorFrame  # noqa: E402
from ssimkit.media import StreamHeader, write_planar_raw, write_pnm, write_report, write_y4m  # noqa: E402
from ssimkit.pipeline import PipelineSpec, expand_preset, run_score  # noqa: E402

from paper_2101_06354_b200 import synth  # noqa: E402

H, W, N = 48, 64, 4

SPECS = {
    "default": lambda: PipelineSpec(SsimConfig()),
    "enhanced": lambda: expand_preset("enhanced"),
    "rect8_pp": lambda: PipelineSpec(SsimConfig(window=WindowSpec.rectangular(8), spatial_pool="pp:ps=10,rs=4",
                                                temporal_pool="hm")),
    "ms_rect5": lambda: PipelineSpec(SsimConfig(window=WindowSpec.rectangular(5),
                                                multiscale=MultiscaleSpec.product(3))),
    "kt2_rect7": lambda: PipelineSpec(SsimConfig(window=WindowSpec.rectangular(7)), kt=2),
    "cw_rect": lambda: PipelineSpec(SsimConfig(window=WindowSpec.rectangular(7), color=ColorModelSpec("cw"))),
    "gauss": lambda: PipelineSpec(SsimConfig(window=WindowSpec.gaussian(1.5))),
}


def frames(seed: int):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(N):
        y = synth.inv_f_noise(rng, H, W, 255.0).astype(np.uint8)
        cb = synth.inv_f_noise(rng, H // 2, W // 2, 255.0).astype(np.uint8)
        cr = synth.inv_f_noise(rng, H // 2, W // 2, 255.0).astype(np.uint8)
        out.append((y, cb, cr))
    return out


def distort(fr, seed: int):
    rng = np.random.default_rng(seed)
    return [tuple(np.clip(p.astype(int) + rng.integers(-18, 19, p.shape), 0, 255).astype(np.uint8) for p in f)
            for f in fr]


def main() -> None:
    out: dict[str, np.ndarray] = {}
    ref, dist = frames(8101), None
    dist = distort(ref, 8102)
    for i, (a, b) in enumerate(zip(ref, dist)):
        for j in range(3):
            out[f"ref/{i}/{j}"] = a[j]
            out[f"dist/{i}/{j}"] = b[j]
    hd = StreamHeader(W, H, (30, 1), "420", 8)
    with tempfile.TemporaryDirectory() as td:
        td = Path(td)
        to_frames = lambda fr: [ColorFrame(f, "ycbcr-bt709", "420", 8) for f in fr]  # noqa: E731
        write_y4m(td / "r.y4m", to_frames(ref), hd)
        write_y4m(td / "d.y4m", to_frames(dist), hd)
        write_planar_raw(td / "r.yuv", to_frames(ref))
        write_planar_raw(td / "d.yuv", to_frames(dist))
        for name, make in SPECS.items():
            res = run_score(td / "r.y4m", td / "d.y4m", make())
            rec = res["records"]
            out[f"run/{name}/score"] = np.array([r["score"] for r in rec])
            out[f"run/{name}/am"] = np.array([np.nan if r["am"] is None else r["am"] for r in rec])
            out[f"run/{name}/l"] = np.array([np.nan if r["l_mean"] is None else r["l_mean"] for r in rec])
            out[f"run/{name}/cs"] = np.array([np.nan if r["cs_mean"] is None else r["cs_mean"] for r in rec])
            s = res["summary"]
            out[f"run/{name}/pooled"] = np.array(s["pooled_score"])
            out[f"run/{name}/mean"] = np.array(s["mean_score"])
            out[f"run/{name}/keys"] = np.array(sorted(k for k in s if k not in ("user_seconds", "timing_source")))
            for fmt in ("jsonl", "csv"):
                out[f"run/{name}/report_{fmt}"] = np.frombuffer(write_report(rec, fmt), dtype=np.uint8)
            print(name, s["pooled_score"])
        raw = run_score(td / "r.yuv", td / "d.yuv", SPECS["default"](), width=W, height=H)
        out["run/raw_default/score"] = np.array([r["score"] for r in raw["records"]])
        # still images: P5 (8-bit) and P6 (16-bit)
        from ssimkit.frames import LumaPlane

        rng = np.random.default_rng(8103)
        g1 = synth.inv_f_noise(rng, H, W, 255.0).astype(np.uint8)
        g2 = np.clip(g1.astype(int) + rng.integers(-10, 11, g1.shape), 0, 255).astype(np.uint8)
        write_pnm(td / "a.pgm", LumaPlane(g1, 8))
        write_pnm(td / "b.pgm", LumaPlane(g2, 8))
        out["pnm/g1"], out["pnm/g2"] = g1, g2
        out["pnm/score"] = np.array(run_score(td / "a.pgm", td / "b.pgm", SPECS["default"]())["records"][0]["score"])
        c1 = np.stack([synth.inv_f_noise(rng, H, W, 65535.0).astype(np.uint16) for _ in range(3)], axis=-1)
        write_pnm(td / "c.ppm", ColorFrame((c1[..., 0], c1[..., 1], c1[..., 2]), "rgb", "444", 16))
        out["pnm/c1"] = c1
        out["pnm/ppm_bytes"] = np.frombuffer((td / "c.ppm").read_bytes(), dtype=np.uint8)
    np.savez_compressed(HERE / "golden_media_v1.npz", **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
