"""Build libssimk.so in-tree with nvcc for sm_100a (no JIT cache, no torch ABI).

Usage: python -m paper_2101_06354_b200.csrc.build  (or build() from __graft_entry__)
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
PKG = HERE.parent
REPO = PKG.parent
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libssimk.so"
SOURCES = ["gauss_ssim.cu", "gauss_generic.cu", "gauss_stride.cu", "gauss_stride_s2.cu", "gauss_stride_s3.cu", "gauss_stride_s4.cu", "gauss_stride_s5.cu", "gauss_stride_s6.cu", "gauss_stride_s7.cu", "gauss_stride_s8.cu", "gauss_u8.cu", "gauss_u16.cu", "gauss_u32.cu", "gauss_f32.cu", "box_ssim.cu",
           "box_block.cu", "volume.cu", "aux_kernels.cu", "pool_adapt.cu", "pool_exact.cu", "color_models.cu", "capi.cu"]
HEADERS = ["common.cuh", "kernels.h", "gauss_ssim.cuh", "gauss_stride.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
         "-Xptxas", "-v", "-I", str(REPO / "include")]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the B200 engine has no CPU fallback")


def _stale(lib: Path = LIB) -> bool:
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    deps = [HERE / s for s in SOURCES + HEADERS] + [REPO / "include" / "ssimk.h"]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, stress: bool = False, variant: str = "",
          defines: tuple = ()) -> Path:
    """stress=True: the synchronisation-stress variant (-DSSK_SYNC_STRESS, random warp delays at
    every barrier hand-off) into _lib/stress/libssimk.so, for tools/sync_stress.py only.
    variant/defines: an A/B build with extra -D flags into _lib/<variant>/libssimk.so."""
    if stress:
        variant, defines = "stress", ("SSK_SYNC_STRESS",)
    lib_out = OUT_DIR / variant / "libssimk.so" if variant else LIB
    if not force and not _stale(lib_out):
        return lib_out
    lib_out.parent.mkdir(parents=True, exist_ok=True)
    obj_dir = OUT_DIR / (f"obj_{variant}" if variant else "obj")
    obj_dir.mkdir(exist_ok=True)
    cc = nvcc()
    extra = [f"-D{d}" for d in defines]

    def obj_stale(src: str, obj: Path) -> bool:
        if force or not obj.exists():
            return True
        deps = [HERE / src, HERE / "common.cuh", HERE / "kernels.h", REPO / "include" / "ssimk.h"]
        if src.startswith("gauss_"):
            deps += [HERE / "gauss_ssim.cuh", HERE / "gauss_stride.cuh"]
        return any(d.stat().st_mtime > obj.stat().st_mtime for d in deps)

    def compile_one(src: str) -> tuple[str, str]:
        obj = obj_dir / (Path(src).stem + ".o")
        if not obj_stale(src, obj):
            return str(obj), ""
        cmd = [cc, *ARCH, *FLAGS, *extra, "-c", str(HERE / src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return str(obj), r.stderr

    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            sys.stderr.write(log)
    tmp = lib_out.with_suffix(".so.tmp")
    cmd = [cc, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib_out)
    return lib_out


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), "")
    defs = tuple(a.split("=", 1)[1] for a in sys.argv if a.startswith("--define="))
    print(build(force="--force" in sys.argv, verbose=True, stress="--stress" in sys.argv, variant=var,
                defines=defs))
