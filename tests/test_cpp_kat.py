"""The reference's known-answer tests, ported to C++ against the drop-in
header include/samo_b200/samo.hpp (tests/cpp/kat_test.cpp).

CPU: the C++ mirror of the reference API compiles and links against
libsamo_cuda.so.  GPU: the KAT binary passes on the device."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "cpp" / "kat_test.cpp"
BIN = ROOT / "tests" / "cpp" / "kat_test"
LIBDIR = ROOT / "paper_2302_05045_b200"


def build_kat() -> Path:
    from paper_2302_05045_b200 import build
    build.build()
    if BIN.exists() and BIN.stat().st_mtime > max(SRC.stat().st_mtime,
                                                  (ROOT / "include/samo_b200/samo.hpp").stat().st_mtime,
                                                  (LIBDIR / "libsamo_cuda.so").stat().st_mtime):
        return BIN
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", f"-I{ROOT / 'include'}",
           "-I/usr/local/cuda/include", str(SRC), "-o", str(BIN),
           f"-L{LIBDIR}", "-lsamo_cuda", "-L/usr/local/cuda/lib64", "-lcudart",
           f"-Wl,-rpath,{LIBDIR}", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return BIN


def test_cpp_mirror_compiles_and_links():
    assert build_kat().exists()


@pytest.mark.gpu
def test_cpp_kats_pass_on_device(cuda):
    exe = build_kat()
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-2000:]
    assert " 0 failed" in res.stdout
