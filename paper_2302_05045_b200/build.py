"""In-tree build of libsamo_cuda.so (sm_100a) — no JIT cache, no setuptools.

    python -m paper_2302_05045_b200.build          # build if stale
    python -m paper_2302_05045_b200.build --force  # rebuild

The shared library is written next to this file so it travels with the repo
snapshot to the GPU box (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libsamo_cuda.so"
CHECKED_LIB = PKG / "libsamo_cuda_checked.so"
SOURCES = ["abi.cu", "model.cu", "dp.cu", "kernels_step.cu", "kernels_fused.cu", "kernels_prune.cu", "kernels_gemm.cu"]
HEADERS = ["common.cuh", "kernels.cuh", "host.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
    "--expt-relaxed-constexpr",
    # Bit-exact IEEE arithmetic: no contraction, no fast math, denormals kept.
    "-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale(lib: Path = None) -> bool:
    lib = lib or LIB
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "samo_cuda.h",
                                                    ROOT / "include" / "samo_cuda_testing.h", Path(__file__)]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> Path:
    """checked: device bounds checks + trapping waits (-DSAMO_CHECKED) into
    libsamo_cuda_checked.so, for test runs with SAMO_LIB pointing at it."""
    lib = CHECKED_LIB if checked else LIB
    if not force and not _stale(lib):
        return lib
    objdir = PKG / ("build_checked" if checked else "build")
    objdir.mkdir(exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = objdir / (Path(src).stem + ".o")
        cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *(["-DSAMO_CHECKED"] if checked else []),
               "-I", str(ROOT / "include"), "-I", str(CSRC), "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        objs.append(str(obj))
    tmp = lib.with_suffix(".so.tmp")
    link = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *objs,
            "-L/usr/lib/x86_64-linux-gnu", "-lnccl", "-cudart", "static",
            "-Xlinker", "--no-undefined"]
    if verbose:
        print(" ".join(link), flush=True)
    subprocess.run(link, check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("--checked", action="store_true", help="device bounds checks (libsamo_cuda_checked.so)")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose, checked=a.checked))
    sys.exit(0)
