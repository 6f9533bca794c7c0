"""The reference's OWN test files, run unmodified against the B200 engine.

tools/install_reference.sh places ssimkit's tests under baseline/_ref/ssimkit_tests (untracked,
like the reference package; the snapshot carries it to the GPU box).  They import
``ssimkit.*``, which tests/refsuite/ssimkit answers from paper_2101_06354_b200, so every
function under test runs on the CUDA path.  Files: the hot-path ★ suites (stats, ssim,
multiscale, color) plus pooling, frames, the acceptance criteria and SSIM-3D.

Failures must be among the ones listed in tests/refsuite/expected_failures.json, each with
its reason (today: two acceptance criteria of subsystems outside the hot path).
"""

import json
import os
import subprocess
import sys
import xml.etree.ElementTree as ET
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

REPO = Path(__file__).resolve().parents[1]
SUITE = REPO / "baseline" / "_ref" / "ssimkit_tests"
FILES = ["test_stats.py", "test_ssim.py", "test_multiscale.py", "test_color.py", "test_pooling.py",
         "test_frames.py", "test_acceptance.py", "test_spatiotemporal.py"]
EXPECTED = json.loads((REPO / "tests" / "refsuite" / "expected_failures.json").read_text())


@pytest.mark.parametrize("name", FILES)
def test_reference_suite_file(cuda, tmp_path, name):
    if not (SUITE / name).exists():
        pytest.skip("reference tests not installed (tools/install_reference.sh)")
    xml = tmp_path / "junit.xml"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(REPO / "tests" / "refsuite"), str(REPO)]))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-o", "addopts=",
                        name, f"--junitxml={xml}"], cwd=SUITE, env=env, capture_output=True, text=True,
                       timeout=900)
    assert xml.exists(), r.stdout[-3000:] + r.stderr[-3000:]
    failed, passed = [], 0
    for case in ET.parse(xml).getroot().iter("testcase"):
        cls = case.get("classname").split(".")[-1]
        tid = f"{name}::{case.get('name')}" if cls == name[:-3] else f"{name}::{cls}::{case.get('name')}"
        if case.find("failure") is not None or case.find("error") is not None:
            failed.append(tid)
        elif case.find("skipped") is None:
            passed += 1
    allowed = {k for k in EXPECTED if k.startswith(name + "::")}
    unexpected = sorted(set(failed) - allowed)
    assert not unexpected, "\n".join(unexpected) + "\n" + r.stdout[-6000:]
    assert passed > 0
