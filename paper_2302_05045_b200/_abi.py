"""ctypes binding of the C ABI in include/samo_cuda.h (libsamo_cuda.so).

The library is the only compute path: there is no CPU fallback, and importing
this module fails loudly when the shared library has not been built.
Status codes are rethrown as the reference's exception classes
(error.hpp:9-36).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libsamo_cuda.so"


class SamoError(RuntimeError):
    status = -1


class DimensionError(SamoError, ValueError):       # error.hpp:9-12
    status = 1


class ParameterError(SamoError, ValueError):       # error.hpp:14-17
    status = 2


class SamoIndexError(SamoError, IndexError):       # error.hpp:19-22
    status = 3


class StateError(SamoError):                       # error.hpp:24-27
    status = 4


class ConfigError(SamoError):                      # error.hpp:29-32
    status = 5


class CudaError(SamoError):
    status = 6


class NcclError(SamoError):
    status = 7


class OutOfDeviceMemory(CudaError):
    status = 8


_BY_STATUS = {c.status: c for c in (DimensionError, ParameterError, SamoIndexError, StateError,
                                    ConfigError, CudaError, NcclError, OutOfDeviceMemory)}

u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p


class OptimizerConfig(C.Structure):
    """samo_optimizer_config == samo::OptimizerConfig (train.hpp:70-87)."""
    _fields_ = [("learning_rate", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float),
                ("epsilon", C.c_float), ("loss_scale", C.c_float), ("weight_decay", C.c_float)]

    def __init__(self, learning_rate=1e-3, beta1=0.9, beta2=0.999, epsilon=1e-8,
                 loss_scale=1024.0, weight_decay=0.0):
        super().__init__(learning_rate, beta1, beta2, epsilon, loss_scale, weight_decay)


class LayerDesc(C.Structure):
    _fields_ = [("dense_len", C.c_uint64), ("nnz", C.c_uint64)]


class LayerView(C.Structure):
    _fields_ = [("theta16", vp), ("theta32", vp), ("adam_m", vp), ("adam_v", vp),
                ("grad32", vp), ("indices", vp), ("dense_len", C.c_uint64),
                ("nnz", C.c_uint64), ("k_offset", C.c_uint64), ("grad16", vp)]


class StepRecord(C.Structure):
    _fields_ = [("t", C.c_uint64), ("skipped_steps", C.c_uint64), ("beta1_pow", C.c_float),
                ("beta2_pow", C.c_float), ("grad_norm", C.c_float), ("last_skipped", C.c_uint32)]


class MemoryReport(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in (
        "dense_params", "kept", "theta16_bytes", "compressed_state_bytes", "index_bytes",
        "table_bytes", "device_bytes", "reference_steady_bytes", "reference_peak_bytes")]


_SIGS = {
    "samo_abi_version": (C.c_int, []),
    "samo_status_string": (C.c_char_p, [C.c_int]),
    "samo_last_error": (C.c_char_p, []),
    "samo_kernel_launch_count": (C.c_uint64, []),
    "samo_float_to_half": (C.c_int, [vp, vp, C.c_uint64, vp]),
    "samo_half_to_float": (C.c_int, [vp, vp, C.c_uint64, vp]),
    "samo_compress_u16": (C.c_int, [vp, C.c_uint64, vp, C.c_uint64, C.c_uint64, vp, vp]),
    "samo_compress_u32": (C.c_int, [vp, C.c_uint64, vp, C.c_uint64, C.c_uint64, vp, vp]),
    "samo_expand_u16": (C.c_int, [vp, C.c_uint64, vp, C.c_uint64, C.c_uint64, C.c_uint64, vp, vp]),
    "samo_expand_u32": (C.c_int, [vp, C.c_uint64, vp, C.c_uint64, C.c_uint64, C.c_uint64, vp, vp]),
    "samo_downcast_expand": (C.c_int, [vp, C.c_uint64, vp, C.c_uint64, vp, vp]),
    "samo_optimizer_config_default": (None, [C.POINTER(OptimizerConfig)]),
    "samo_optimizer_config_validate": (C.c_int, [C.POINTER(OptimizerConfig)]),
    "samo_adam_update": (C.c_int, [vp, vp, vp, vp, C.c_uint64, C.POINTER(OptimizerConfig),
                                   C.c_float, C.c_float, vp]),
    "samo_unpruned_count": (C.c_uint64, [C.c_double, C.c_uint64]),
    "samo_magnitude_prune": (C.c_int, [C.POINTER(vp), u64p, u8p, C.c_int, C.c_double, C.c_int,
                                       C.POINTER(vp), u64p, vp]),
    "samo_comm_unique_id": (C.c_int, [u8p]),
    "samo_comm_create": (C.c_int, [u8p, C.c_int, C.c_int, C.POINTER(vp)]),
    "samo_comm_destroy": (C.c_int, [vp]),
    "samo_comm_size": (C.c_int, [vp]),
    "samo_allreduce_sum_f32": (C.c_int, [vp, vp, C.c_uint64, vp]),
    "samo_model_create": (C.c_int, [C.POINTER(LayerDesc), C.c_int, C.c_uint32, C.POINTER(vp)]),
    "samo_model_destroy": (C.c_int, [vp]),
    "samo_model_num_layers": (C.c_int, [vp]),
    "samo_model_layer_view": (C.c_int, [vp, C.c_int, C.POINTER(LayerView)]),
    "samo_model_totals": (C.c_int, [vp, u64p, u64p, u64p]),
    "samo_model_device_bytes": (C.c_uint64, [vp]),
    "samo_model_set_indices": (C.c_int, [vp, C.c_int, vp, C.c_uint64, C.c_int, vp]),
    "samo_model_finalize": (C.c_int, [vp, vp]),
    "samo_model_init_layer": (C.c_int, [vp, C.c_int, vp, C.c_uint64, vp]),
    "samo_model_set_config": (C.c_int, [vp, C.POINTER(OptimizerConfig)]),
    "samo_model_set_grad_dtype": (C.c_int, [vp, C.c_int]),
    "samo_model_grad_dtype": (C.c_int, [vp]),
    "samo_model_attach_comm": (C.c_int, [vp, vp]),
    "samo_model_set_exchange": (C.c_int, [vp, C.c_int]),
    "samo_model_exchange_mode": (C.c_int, [vp]),
    "samo_model_shard_layout": (C.c_int, [vp, u64p, u64p, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "samo_model_enable_phase_timing": (C.c_int, [vp, C.c_int]),
    "samo_model_phase_times": (C.c_int, [vp, C.POINTER(C.c_float), C.c_int]),
    "samo_model_set_grads": (C.c_int, [vp, C.POINTER(vp), vp]),
    "samo_model_gather": (C.c_int, [vp, vp]),
    "samo_model_sink_dense": (C.c_int, [vp, C.c_int, vp, vp]),
    "samo_model_p2p_features": (C.c_int, [vp]),
    "samo_model_attach_local_group": (C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
    "samo_local_group_step": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, vp]),
    "samo_local_group_step_sunk": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, vp]),
    "samo_model_step_sunk": (C.c_int, [vp, vp]),
    "samo_model_sink_dw": (C.c_int, [vp, C.c_int, vp, vp, C.c_uint64, C.c_uint64, C.c_uint64, vp]),
    "samo_dw_gemm_f16": (C.c_int, [vp, vp, C.c_uint64, C.c_uint64, C.c_uint64, vp, vp]),
    "samo_model_exchange": (C.c_int, [vp, vp]),
    "samo_model_update": (C.c_int, [vp, vp]),
    "samo_model_step": (C.c_int, [vp, vp]),
    "samo_model_step_graph": (C.c_int, [vp, vp]),
    "samo_model_step_record": (C.c_int, [vp, C.POINTER(StepRecord), vp]),
    "samo_model_step_record_async": (C.c_int, [vp, vp, vp]),
    "samo_model_set_step_record": (C.c_int, [vp, C.POINTER(StepRecord), vp]),
    "samo_model_check_invariants": (C.c_int, [vp, vp]),
    "samo_model_save": (C.c_int, [vp, C.c_char_p, vp]),
    "samo_model_load": (C.c_int, [C.c_char_p, C.c_uint32, C.POINTER(vp), vp]),
    "samo_model_memory": (C.c_int, [vp, C.POINTER(MemoryReport)]),
    "samo_copy_async": (C.c_int, [vp, vp, C.c_uint64, vp]),
    "samo_stream_synchronize": (C.c_int, [vp]),
    "samo_synth_uniform_f32": (C.c_int, [vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_float, vp]),
    "samo_synth_uniform_f16": (C.c_int, [vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_float,
                                         C.c_float, vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(path: os.PathLike | str | None = None) -> C.CDLL:
    """Loads libsamo_cuda.so (once) and declares every ABI signature."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else Path(os.environ.get("SAMO_LIB", LIB_PATH))
    if not p.exists():
        raise ImportError(
            f"{p} is missing: build it with `python -m paper_2302_05045_b200.build` "
            "(the SAMO path has no CPU fallback)")
    try:  # torch first: its bundled libnccl.so.2 (newer than the system one) then
        import torch  # noqa: F401  serves our NCCL dependency, and torch stays importable
    except ImportError:
        pass
    lib = C.CDLL(str(p))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(status: int) -> None:
    if status == 0:
        return
    lib = load()
    msg = (lib.samo_last_error() or b"").decode()
    raise _BY_STATUS.get(status, SamoError)(f"[{lib.samo_status_string(status).decode()}] {msg}")


def call(name: str, *args) -> int:
    rc = getattr(load(), name)(*args)
    check(rc)
    return rc
