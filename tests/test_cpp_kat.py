"""The reference's known-answer tests against the drop-in C++ mirror
(include/samo_b200/samo.hpp, reached through the reference's own header names
include/samo/*.hpp):

* tests/cpp/kat_test.cpp — the reference KATs ported (half, prune, store,
  Adam, the SamoTrainer OptimizerStep tests of train_test.cpp:139-199);
* the reference's UNMODIFIED proj/tests/store_test.cpp, compiled from
  /root/reference against the mirror with only the include path changed
  (GoogleTest is absent: tests/cpp/gtest_shim provides the macros); the
  binary is built here and travels to the GPU box under tests/cpp/_ref/;
* tests/cpp/half_host_test.cpp — the mirror's host Half conversions over all
  2^32 floats and 65,536 halves against the pinned oracle (CPU).

CPU: everything compiles and links against libsamo_cuda.so; the host Half
check runs.  GPU: the KAT binary and the reference store_test pass."""
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
    if _newer(BIN, [SRC, *HEADERS, LIBDIR / "libsamo_cuda.so"]):
        return BIN
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", f"-I{ROOT / 'include'}",
           "-I/usr/local/cuda/include", str(SRC), "-o", str(BIN),
           f"-L{LIBDIR}", "-lsamo_cuda", "-L/usr/local/cuda/lib64", "-lcudart",
           f"-Wl,-rpath,{LIBDIR}", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return BIN


REF_TESTS = Path("/root/reference/proj/tests")
REF_BIN_DIR = ROOT / "tests" / "cpp" / "_ref"
HEADERS = [ROOT / "include/samo_b200/samo.hpp", *sorted((ROOT / "include/samo").glob("*.hpp")),
           ROOT / "tests/cpp/gtest_shim/gtest/gtest.h"]


def _newer(target: Path, deps) -> bool:
    return target.exists() and target.stat().st_mtime > max(d.stat().st_mtime for d in deps)


def build_ref_store_test() -> Path | None:
    """The reference's store_test.cpp against the mirror (None when neither
    the reference sources nor a prebuilt binary are present)."""
    exe = REF_BIN_DIR / "store_test"
    src = REF_TESTS / "store_test.cpp"
    if not src.exists():
        return exe if exe.exists() else None
    from paper_2302_05045_b200 import build
    build.build()
    if _newer(exe, [src, *HEADERS, LIBDIR / "libsamo_cuda.so"]):
        return exe
    REF_BIN_DIR.mkdir(parents=True, exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", f"-I{ROOT / 'tests/cpp/gtest_shim'}",
           "-I/usr/local/cuda/include", str(src), "-o", str(exe),
           f"-L{LIBDIR}", "-lsamo_cuda", "-L/usr/local/cuda/lib64", "-lcudart",
           f"-Wl,-rpath,{LIBDIR}", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_host_half_conversions_exhaustive(oracle):
    exe = ROOT / "tests" / "cpp" / "half_host_test"
    src = ROOT / "tests" / "cpp" / "half_host_test.cpp"
    if not _newer(exe, [src, ROOT / "include/samo_b200/samo.hpp"]):
        subprocess.run(["g++", "-std=c++20", "-O2", "-fopenmp", f"-I{ROOT / 'include'}",
                        "-I/usr/local/cuda/include", str(src), "-o", str(exe),
                        f"-L{ROOT / 'oracle'}", "-loracle", f"-Wl,-rpath,{ROOT / 'oracle'}"],
                       check=True, capture_output=True, text=True)
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "mismatches: 0 of 4294967296" in res.stdout and "mismatches: 0 of 65536" in res.stdout


def test_reference_store_test_compiles_against_mirror():
    if not (REF_TESTS / "store_test.cpp").exists():
        pytest.skip("reference sources not present (built where they are)")
    assert build_ref_store_test().exists()


def test_reference_store_test_host_suites_on_cpu():
    """The host-arithmetic suites of the reference's store_test.cpp
    (MemoryModel's Rational arithmetic and analytical model, the empty-model
    measured_bytes) run without a GPU; the rest needs the device."""
    exe = build_ref_store_test()
    if exe is None:
        pytest.skip("no reference store_test binary")
    res = subprocess.run([str(exe), "--gtest_filter=MemoryModel.PaperEndpoints:MemoryModel.ReportIdentities:"
                          "MemoryModel.Savings*:MeasuredBytes.EmptyModel"],
                         capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]
    assert "4 tests, 4 passed, 0 failed" in res.stdout, res.stdout[-2000:]


@pytest.mark.gpu
def test_reference_store_test_passes_on_device(cuda):
    exe = build_ref_store_test()
    if exe is None:
        pytest.skip("no reference store_test binary (build it where /root/reference exists)")
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-2000:]
    assert " 0 failed" in res.stdout


def test_cpp_mirror_compiles_and_links():
    assert build_kat().exists()


@pytest.mark.gpu
def test_cpp_kats_pass_on_device(cuda):
    exe = build_kat()
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-2000:]
    assert " 0 failed" in res.stdout
