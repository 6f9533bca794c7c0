"""The C-ABI library loads without a GPU and exports exactly what include/ssimk.h declares."""

import ctypes
import re
import shutil
import subprocess
from pathlib import Path

import pytest

from paper_2101_06354_b200 import _native as nat

REPO = Path(__file__).resolve().parents[1]
HEADER = REPO / "include" / "ssimk.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(ssk_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = nat.load_library()
    names = declared_functions()
    assert names, "no declarations parsed"
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing
    assert sorted(nat.EXPORTED_SYMBOLS) == names
    # the symbols must be exported with C linkage (no mangling)
    nm = shutil.which("nm")
    if nm:
        out = subprocess.run([nm, "-D", "--defined-only", str(nat.LIB_PATH)], capture_output=True, text=True).stdout
        exported = set(re.findall(r"\bT (ssk_\w+)", out))
        assert set(names) <= exported


def test_abi_version_and_errors():
    lib = nat.load_library()
    assert lib.ssk_abi_version() == nat.ABI_VERSION
    assert lib.ssk_strerror(0) == b"ok"
    assert b"window" in lib.ssk_strerror(nat.E_WINDOW)
    assert lib.ssk_strerror(-99) == b"unknown error"


def test_argument_errors_need_no_gpu():
    """Validation happens before any launch, so bad calls fail cleanly even on a CPU host."""
    lib = nat.load_library()
    assert lib.ssk_ssim(None, None, 1, None, None, None, 0, None) == nat.E_ARG
    p = nat.Planes(ref=16, dist=32, dtype=nat.U8, n=1, h=8, w=8, bit_depth=8, row_pitch=16, frame_pitch=128)
    win = nat.Window(shape=nat.RECT, k=11, stride=1, c1=1.0, c2=1.0)
    sums = ctypes.c_void_p(64)
    assert lib.ssk_ssim(ctypes.byref(p), ctypes.byref(win), 1, sums, None, None, 0, None) == nat.E_WINDOW
    win.k = 4
    assert lib.ssk_ssim(ctypes.byref(p), ctypes.byref(win), 1, sums, None, None, 0, None) == nat.E_WORKSPACE
    p.ref = 17  # misaligned
    assert lib.ssk_ssim(ctypes.byref(p), ctypes.byref(win), 1, sums, None, None, 0, None) == nat.E_ALIGN
    p.ref = 16
    win.shape, win.k = nat.GAUSS, 4  # even Gaussian window
    assert lib.ssk_ssim(ctypes.byref(p), ctypes.byref(win), 1, sums, None, None, 0, None) == nat.E_SHAPE
    assert lib.ssk_ssim_workspace_bytes(ctypes.byref(p), ctypes.byref(win)) == 0
    win.shape, win.k = nat.RECT, 3
    assert lib.ssk_ssim_workspace_bytes(ctypes.byref(p), ctypes.byref(win)) > 0
    means = ctypes.c_void_p(64)
    assert lib.ssk_msssim(ctypes.byref(p), ctypes.byref(win), 3, None, 0, means, None, None, None, 0,
                          None) == nat.E_LEVELS


def test_error_codes_map_to_reference_exceptions():
    from paper_2101_06354_b200 import errors

    with pytest.raises(errors.WindowLargerThanImage):
        nat.raise_for(nat.E_WINDOW)
    with pytest.raises(errors.TooManyLevels):
        nat.raise_for(nat.E_LEVELS)
    with pytest.raises(errors.TooSmall):
        nat.raise_for(nat.E_TOO_SMALL)
    with pytest.raises(errors.ValidationError):
        nat.raise_for(nat.E_ARG)


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_ctypes_struct_layout_matches_header(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "ssimk.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu %zu\\n\", sizeof(ssk_planes), offsetof(ssk_planes,row_pitch),"
        " offsetof(ssk_planes,frame_pitch), sizeof(ssk_window), offsetof(ssk_window,c1), offsetof(ssk_window,taps));"
        "printf(\"%zu\\n\", offsetof(ssk_window,sigma));"
        "return 0;}\n"
    )
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", str(REPO / "include"), str(src), "-o", str(exe)], check=True)
    vals = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert vals == [
        ctypes.sizeof(nat.Planes), nat.Planes.row_pitch.offset, nat.Planes.frame_pitch.offset,
        ctypes.sizeof(nat.Window), nat.Window.c1.offset, nat.Window.taps.offset, nat.Window.sigma.offset,
    ]


def _gauss_call(win, h=64, w=64):
    lib = nat.load_library()
    pitch = (w + 15) // 16 * 16
    p = nat.Planes(ref=256, dist=512, dtype=nat.U8, n=1, h=h, w=w, bit_depth=8, row_pitch=pitch,
                   frame_pitch=pitch * h)
    return lib.ssk_ssim_workspace_bytes(ctypes.byref(p), ctypes.byref(win))


def _gauss_window(k=11, sigma=0.0, taps=None):
    win = nat.Window(shape=nat.GAUSS, k=k, stride=1, c1=6.5025, c2=58.5225, sigma=sigma)
    for i, t in enumerate(taps if taps is not None else []):
        win.taps[i] = float(t)
    return win


def test_gaussian_window_taps_are_validated():
    """ABI v9: a Gaussian window needs sigma or valid taps.  Zero taps without sigma (a binding
    that forgot them), negative, asymmetric or unnormalised taps are rejected (planning
    fails -> workspace query 0 / SSK_E_ARG) instead of silently scoring q = 1."""
    good = nat.gaussian_taps(1.5, 11)
    assert _gauss_call(_gauss_window(taps=good)) > 0
    assert _gauss_call(_gauss_window(sigma=1.5)) > 0            # library builds the taps
    assert _gauss_call(_gauss_window()) == 0                     # neither
    asym = good.copy()
    asym[0] *= 1.01
    asym /= asym.sum()
    assert _gauss_call(_gauss_window(taps=asym)) == 0
    assert _gauss_call(_gauss_window(taps=good * 2.0)) == 0      # not normalised
    neg = good.copy()
    neg[0] = neg[-1] = -neg[0]
    assert _gauss_call(_gauss_window(taps=neg)) == 0
    extra = list(good) + [0.01]                                  # non-zero past k
    assert _gauss_call(_gauss_window(taps=extra)) == 0
    assert _gauss_call(_gauss_window(sigma=-1.0)) == 0
    lib = nat.load_library()
    p = nat.Planes(ref=256, dist=512, dtype=nat.U8, n=1, h=64, w=64, bit_depth=8, row_pitch=64, frame_pitch=4096)
    rc = lib.ssk_ssim(ctypes.byref(p), ctypes.byref(_gauss_window()), 1, ctypes.c_void_p(64), None, None, 0, None)
    assert rc == nat.E_ARG


def test_wide_gaussian_windows_plan_with_sigma():
    """k > 31 (sigma > 5 at the default size): planned on the generic kernel from sigma alone;
    taps cannot carry them; k above SSK_GAUSS_MAX_K is a shape error."""
    from paper_2101_06354_b200.options import WindowSpec

    w37 = nat.make_window(WindowSpec.gaussian(6.0), 6.5025, 58.5225)
    assert w37.k == 37 and w37.sigma == 6.0 and all(t == 0.0 for t in w37.taps)
    assert _gauss_call(w37, 200, 300) > 0
    assert _gauss_call(_gauss_window(k=37), 200, 300) == 0       # no sigma
    assert _gauss_call(_gauss_window(k=257, sigma=40.0), 300, 300) == 0
    assert _gauss_call(_gauss_window(k=255, sigma=40.0), 300, 300) > 0
    assert _gauss_call(_gauss_window(k=37, sigma=6.0), 30, 300) == 0   # window larger than image


def build_c_cli(out_dir):
    """Compile tests/c_abi/ssim_cli.c -- a host program using only the C ABI -- with gcc."""
    exe = Path(out_dir) / "ssim_cli"
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Werror", "-I", str(REPO / "include"), "-I", "/usr/local/cuda/include",
           str(REPO / "tests" / "c_abi" / "ssim_cli.c"), "-o", str(exe), "-L", str(nat.LIB_PATH.parent), "-lssimk",
           f"-Wl,-rpath,{nat.LIB_PATH.parent}", "-L", "/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


@pytest.mark.skipif(shutil.which("gcc") is None or not Path("/usr/local/cuda/include/cuda_runtime.h").exists(),
                    reason="needs gcc and the CUDA headers")
def test_c_host_program_compiles_against_the_abi(tmp_path):
    """include/ssimk.h is plain C99 and libssimk.so links into a C program (no C++, no torch)."""
    exe = build_c_cli(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 1 and "usage" in r.stderr


def test_round2_entry_points_validate_without_gpu():
    """The r2 C-ABI additions reject bad arguments before any launch (no GPU needed)."""
    lib = nat.load_library()
    vp = ctypes.c_void_p
    assert lib.ssk_stats_from_sums(None, None, None, None, None, 4, 1.0, None, None) == nat.E_ARG
    assert lib.ssk_stats_from_sums(vp(8), vp(8), vp(8), vp(8), vp(8), 4, 0.0, vp(8), None) == nat.E_ARG  # area
    assert lib.ssk_term_maps(None, vp(8), vp(8), vp(8), vp(8), 4, 1.0, 1.0, vp(8), None) == nat.E_ARG
    assert lib.ssk_divide(None, 4, 2.0, vp(8), None) == nat.E_ARG
    m = nat.Maps(values=256, aux=None, dtype=nat.F64, n=1, h=4, w=5, row_pitch=5, frame_pitch=20,
                 aux_row_pitch=0, aux_frame_pitch=0)
    ws = lib.ssk_pairwise_workspace_bytes(ctypes.byref(m))
    assert ws == 8  # 20 samples: a single subtree
    out = vp(64)
    assert lib.ssk_pairwise_sum(ctypes.byref(m), nat.PW_SQDEV, 0.0, 0.0, 0.0, None, out, vp(64), ws, None) == nat.E_ARG
    assert lib.ssk_pairwise_sum(ctypes.byref(m), 99, 0.0, 0.0, 0.0, None, out, vp(64), ws, None) == nat.E_ARG
    assert lib.ssk_pairwise_sum(ctypes.byref(m), nat.PW_LW, 0.0, 0.0, 0.0, None, out, vp(64), ws, None) == nat.E_ARG
    assert lib.ssk_pairwise_sum(ctypes.byref(m), nat.PW_V, 0.0, 0.0, 0.0, None, out, vp(64), 0, None) == \
        nat.E_WORKSPACE
    big = nat.Maps(values=256, aux=None, dtype=nat.F64, n=2, h=1070, w=1910, row_pitch=1910,
                   frame_pitch=1070 * 1910, aux_row_pitch=0, aux_frame_pitch=0)
    assert lib.ssk_pairwise_workspace_bytes(ctypes.byref(big)) == 2 * (1 << 12) * 8  # depth-12 top tree
