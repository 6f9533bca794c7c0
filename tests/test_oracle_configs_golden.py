"""CPU: the synthetic generators and the oracle against the reference's full-size config goldens.

golden_configs_v1.npz holds ssimkit's own scores (tests/golden/make_golden_configs.py); here
the frames are regenerated (CRC-checked) and a sample of them is re-scored by the oracle,
pinning the oracle at the configurations' stated sizes.  The GPU tests
(tests/test_gpu_configs.py) compare the engine against the same goldens on every frame.
"""

import zlib
from pathlib import Path

import numpy as np
import pytest

from oracle import ssim_oracle as O
from paper_2101_06354_b200 import synth

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden_configs_v1.npz"
WIN = dict(shape="gauss", k=11, sigma=1.5)


@pytest.fixture(scope="module")
def gold():
    with np.load(GOLDEN) as z:
        return {k: z[k] for k in z.files}


def crc(*arrays):
    c = 0
    for a in arrays:
        c = zlib.crc32(np.ascontiguousarray(a).tobytes(), c)
    return c


def test_config2_frame0_oracle_matches_reference(gold):
    a, b = synth.dct_pair(2, 0)
    assert crc(a, b) == gold["c2/crc"][0]
    lv = O.scale_scores(a, b, 5, **WIN)
    assert np.max(np.abs(np.array(lv) - gold["c2/levels"][0])) < 1e-12
    assert abs(O.combine_scale_scores(lv, "product", O.STANDARD_EXPONENTS) - gold["c2/msssim"][0]) < 1e-12
    assert np.max(np.abs(np.array(O.ssim_terms(a, b, **WIN)) - gold["c2/terms"][0])) < 1e-12


def test_config3_first_and_last_frame(gold):
    vid = synth.VideoConfig3()
    wts = tuple(gold["c3/weights"])
    for t in (0, 299):
        r, d = vid.pair(t)
        assert crc(*r, *d) == gold["c3/crc"][t]
        ch = O.channel_scores(r, d, **WIN)
        assert np.max(np.abs(np.array(ch) - gold["c3/planes"][t])) < 1e-12
        assert abs(O.fixed_weight(ch, wts) - gold["c3/scores"][t]) < 1e-12
    assert abs(O.pool_temporal_am(gold["c3/scores"]) - float(gold["c3/pooled"])) < 1e-15


def test_config4_pair0_exact_box(gold):
    a, b = synth.config4_pair(0)
    assert crc(a, b) == gold["c4/crc"][0]
    t = O.ssim_terms(a, b, shape="rect", k=8, stride=4, bit_depth=10)
    assert np.max(np.abs(np.array(t) - gold["c4/terms"][0])) < 1e-13
