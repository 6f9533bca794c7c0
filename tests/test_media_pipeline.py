"""File pipeline (run_score), media readers and the report writer vs the reference's outputs.

Golden vectors: tests/golden/golden_media_v1.npz (tests/golden/make_golden_media.py
ran ssimkit's own run_score / write_report / write_pnm).  The media files are
rewritten here from the stored frames.
"""

from pathlib import Path

import numpy as np
import pytest

import paper_2101_06354_b200 as P

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden_media_v1.npz"
H, W, N = 48, 64, 4
SPECS = {
    "default": lambda: P.PipelineSpec(P.SsimConfig()),
    "enhanced": lambda: P.expand_preset("enhanced"),
    "rect8_pp": lambda: P.PipelineSpec(P.SsimConfig(window=P.WindowSpec.rectangular(8), spatial_pool="pp:ps=10,rs=4",
                                                    temporal_pool="hm")),
    "ms_rect5": lambda: P.PipelineSpec(P.SsimConfig(window=P.WindowSpec.rectangular(5),
                                                    multiscale=P.MultiscaleSpec.product(3))),
    "kt2_rect7": lambda: P.PipelineSpec(P.SsimConfig(window=P.WindowSpec.rectangular(7)), kt=2),
    "cw_rect": lambda: P.PipelineSpec(P.SsimConfig(window=P.WindowSpec.rectangular(7), color=P.ColorModelSpec("cw"))),
    "gauss": lambda: P.PipelineSpec(P.SsimConfig(window=P.WindowSpec.gaussian(1.5))),
}


@pytest.fixture(scope="module")
def gmedia():
    with np.load(GOLDEN) as z:
        return {k: z[k] for k in z.files}


def _records(g, name):
    def opt(x):
        return None if np.isnan(x) else float(x)

    return [{"frame": i, "score": float(g[f"run/{name}/score"][i]), "am": opt(g[f"run/{name}/am"][i]),
             "l_mean": opt(g[f"run/{name}/l"][i]), "cs_mean": opt(g[f"run/{name}/cs"][i])}
            for i in range(len(g[f"run/{name}/score"]))]


@pytest.mark.parametrize("name", sorted(SPECS))
def test_report_writer_bytes(gmedia, name):
    """write_report reproduces the reference's jsonl / csv bytes for the reference's records."""
    recs = _records(gmedia, name)
    for fmt in ("jsonl", "csv"):
        assert P.write_report(recs, fmt) == gmedia[f"run/{name}/report_{fmt}"].tobytes()
    from paper_2101_06354_b200 import errors as E

    with pytest.raises(E.ValidationError):
        P.write_report([], "jsonl")


def test_pnm_reader(gmedia, tmp_path):
    p = tmp_path / "c.ppm"
    p.write_bytes(gmedia["pnm/ppm_bytes"].tobytes())
    img = P.read_pnm(p)
    assert img.bit_depth == 16 and img.space == "rgb"
    assert np.array_equal(np.stack(img.channels, axis=-1), gmedia["pnm/c1"])
    (tmp_path / "bad.pgm").write_bytes(b"P5 4 4 70000\n" + b"\0" * 32)
    from paper_2101_06354_b200 import errors as E

    with pytest.raises(E.UnsupportedMaxval):
        P.read_pnm(tmp_path / "bad.pgm")


def _write_streams(g, d):
    ref = [tuple(g[f"ref/{i}/{j}"] for j in range(3)) for i in range(N)]
    dist = [tuple(g[f"dist/{i}/{j}"] for j in range(3)) for i in range(N)]
    P.write_y4m(d / "r.y4m", ref, W, H)
    P.write_y4m(d / "d.y4m", dist, W, H)
    P.write_planar_raw(d / "r.yuv", ref)
    P.write_planar_raw(d / "d.yuv", dist)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(SPECS))
def test_run_score_vs_reference(cuda, gmedia, tmp_path, name):
    _write_streams(gmedia, tmp_path)
    res = P.run_score(tmp_path / "r.y4m", tmp_path / "d.y4m", SPECS[name]())
    tol = 1e-5 if name == "gauss" else 1e-9
    got = np.array([r["score"] for r in res["records"]])
    assert np.allclose(got, gmedia[f"run/{name}/score"], rtol=0, atol=tol)
    for key, col in (("am", "am"), ("l_mean", "l"), ("cs_mean", "cs")):
        vals = np.array([np.nan if r[key] is None else r[key] for r in res["records"]])
        assert np.allclose(vals, gmedia[f"run/{name}/{col}"], rtol=0, atol=tol, equal_nan=True)
    s = res["summary"]
    assert abs(s["pooled_score"] - float(gmedia[f"run/{name}/pooled"])) < tol
    assert sorted(k for k in s if k not in ("user_seconds", "timing_source")) == list(gmedia[f"run/{name}/keys"])
    if name != "gauss":  # 9-significant-digit reports match byte for byte on the exact paths
        assert P.write_report(res["records"], "csv") == gmedia[f"run/{name}/report_csv"].tobytes()


@pytest.mark.gpu
def test_run_score_raw_and_pnm(cuda, gmedia, tmp_path):
    _write_streams(gmedia, tmp_path)
    raw = P.run_score(tmp_path / "r.yuv", tmp_path / "d.yuv", SPECS["default"](), width=W, height=H)
    assert np.allclose([r["score"] for r in raw["records"]], gmedia["run/raw_default/score"], rtol=0, atol=1e-12)
    from paper_2101_06354_b200 import errors as E

    with pytest.raises(E.ValidationError):
        P.run_score(tmp_path / "r.yuv", tmp_path / "d.yuv", SPECS["default"]())
    (tmp_path / "a.pgm").write_bytes(b"P5\n%d %d\n255\n" % (W, H) + gmedia["pnm/g1"].tobytes())
    (tmp_path / "b.pgm").write_bytes(b"P5\n%d %d\n255\n" % (W, H) + gmedia["pnm/g2"].tobytes())
    res = P.run_score(tmp_path / "a.pgm", tmp_path / "b.pgm", SPECS["default"]())
    assert abs(res["records"][0]["score"] - float(gmedia["pnm/score"])) < 1e-12
