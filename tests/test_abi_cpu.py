"""CPU: the C-ABI library is built for sm_100a, loads, and exports every
symbol include/samo_cuda.h declares; without a GPU it refuses to compute
(no CPU fallback) instead of silently doing something else."""
from __future__ import annotations

import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "samo_cuda.h"
TESTING = ROOT / "include" / "samo_cuda_testing.h"  # test harness, outside the boundary


def declared_functions(headers=(HEADER, TESTING)) -> list[str]:
    out = set()
    for h in headers:
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        out |= set(re.findall(r"\b(samo_[a-z0-9_]+)\s*\(", text))
    return sorted(out)


def test_boundary_header_has_no_test_harness():
    product = declared_functions((HEADER,))
    assert "samo_local_group_step" not in product and "samo_model_attach_local_group" not in product
    assert {"samo_local_group_step", "samo_model_attach_local_group"} <= set(declared_functions((TESTING,)))


@pytest.fixture(scope="module")
def lib():
    from paper_2302_05045_b200 import _abi, build
    build.build()
    return _abi.load()


def test_header_declares_the_path():
    fns = declared_functions()
    for must in ("samo_compress_u16", "samo_expand_u16", "samo_adam_update",
                 "samo_magnitude_prune", "samo_model_step", "samo_allreduce_sum_f32"):
        assert must in fns


def test_library_exports_every_declared_symbol(lib):
    so = Path(lib._name)
    out = subprocess.run(["nm", "-D", "--defined-only", str(so)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (samo_[a-z0-9_]+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing


def test_python_binding_covers_header(lib):
    from paper_2302_05045_b200 import _abi
    assert set(declared_functions()) == set(_abi.EXPORTED)


def test_library_is_sm100a(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib._name],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib._name],
                          capture_output=True, text=True).stdout
    assert "UBLKCP" in sass  # 1-D TMA bulk copies in the gather / expand kernels


def test_status_strings(lib):
    assert lib.samo_abi_version() == 1
    names = [lib.samo_status_string(i).decode() for i in range(9)]
    assert names[1:6] == ["DimensionError", "ParameterError", "IndexError", "StateError",
                          "ConfigError"]


def test_host_only_entry_points(lib):
    # prune.hpp:76-79 rounding convention, evaluated on the host in double
    assert lib.samo_unpruned_count(0.9, 16777216) == 1677722
    assert lib.samo_unpruned_count(0.3, 5) == 4
    from paper_2302_05045_b200._abi import OptimizerConfig
    cfg = OptimizerConfig()
    lib.samo_optimizer_config_default(C.byref(cfg))
    assert cfg.learning_rate == C.c_float(1e-3).value and cfg.loss_scale == 1024.0
    assert lib.samo_optimizer_config_validate(C.byref(cfg)) == 0
    cfg.loss_scale = 3.0
    assert lib.samo_optimizer_config_validate(C.byref(cfg)) == 2


def test_no_cpu_fallback(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    from paper_2302_05045_b200._abi import LayerDesc
    d = (LayerDesc * 1)(LayerDesc(16, 4))
    assert lib.samo_model_create(d, 1, 0, C.byref(h)) == 6  # SAMO_E_CUDA
    assert b"no CPU fallback" in lib.samo_last_error()


def test_index_set_widening():
    """uint32 indices >= 2^31 live in int32 tensors as negative values;
    as_int64 widens them without sign extension (dense_len < 2^32)."""
    torch = pytest.importorskip("torch")
    from paper_2302_05045_b200 import samo
    raw = torch.tensor([0, 5, 2**31 - 1, 2**31, 2**32 - 2], dtype=torch.int64).to(torch.int32)
    s = samo.PrunedIndexSet("big", 2**32 - 1, raw)
    assert s.as_int64().tolist() == [0, 5, 2**31 - 1, 2**31, 2**32 - 2]
    assert s.count() == 5


def test_header_is_plain_c99(tmp_path):
    """cgo / JNI / ctypes hosts include the ABI header as C: it must compile as
    strict C99 without warnings."""
    import shutil
    if not shutil.which("gcc"):
        pytest.skip("no gcc")
    src = tmp_path / "h.c"
    src.write_text('#include "samo_cuda.h"\n#include "samo_cuda_testing.h"\nint main(void) { return 0; }\n')
    res = subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I", str(HEADER.parent),
                          "-fsyntax-only", str(src)], capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
