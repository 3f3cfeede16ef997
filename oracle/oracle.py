"""TEST INFRASTRUCTURE ONLY — numpy front-end of the CPU oracle.

`Oracle`  : the C restatement oracle/samo_oracle.c (liboracle.so).
`RefLib`  : the unmodified reference headers behind oracle/ref_shim.cpp
            (oracle/_ref/libsamo_ref.so), when it has been built.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may import
this module; the product path (paper_2302_05045_b200/) never does.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libsamo_ref.so"

vp = C.c_void_p
u64 = C.c_uint64


def build(force: bool = False) -> None:
    """Runs oracle/Makefile (liboracle.so; _ref/ only when /root/reference exists)."""
    if force or not ORACLE_SO.exists() or (
            ORACLE_SO.stat().st_mtime < (HERE / "samo_oracle.c").stat().st_mtime):
        subprocess.run(["make", "-s", "-C", str(HERE), str(ORACLE_SO)], check=True)
    if Path("/root/reference/proj/include/samo").is_dir() and (
            force or not REF_SO.exists()
            or REF_SO.stat().st_mtime < (HERE / "ref_shim.cpp").stat().st_mtime):
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)


def _p(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


def _ptr_array(arrs) -> C.Array:
    return (C.c_void_p * max(1, len(arrs)))(*[a.ctypes.data for a in arrs])


class Cfg(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float),
                ("eps", C.c_float), ("loss_scale", C.c_float), ("wd", C.c_float)]

    def __init__(self, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, loss_scale=1024.0, wd=0.0):
        super().__init__(lr, beta1, beta2, eps, loss_scale, wd)


class StepState(C.Structure):
    _fields_ = [("t", C.c_uint64), ("skipped", C.c_uint64), ("beta1_pow", C.c_float),
                ("beta2_pow", C.c_float), ("grad_norm", C.c_float), ("last_skipped", C.c_uint32)]

    def __init__(self):
        super().__init__(0, 0, 1.0, 1.0, 0.0, 0)


class MT64(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("mti", C.c_int)]


class Oracle:
    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            build()
        lib = C.CDLL(str(path))
        self.lib = lib
        lib.or_float_to_half.restype = C.c_uint16
        lib.or_float_to_half.argtypes = [C.c_float]
        lib.or_half_to_float.restype = C.c_float
        lib.or_half_to_float.argtypes = [C.c_uint16]
        for n in ("or_f2h", "or_h2f"):
            getattr(lib, n).argtypes = [vp, vp, u64]
        for n in ("or_compress_u16", "or_compress_u32"):
            getattr(lib, n).argtypes = [vp, u64, vp, u64, u64, vp]
        for n in ("or_expand_u16", "or_expand_u32"):
            getattr(lib, n).argtypes = [vp, u64, vp, u64, u64, u64, vp]
        lib.or_adam_update.argtypes = [vp, vp, vp, vp, u64, C.POINTER(Cfg), C.c_float, C.c_float]
        lib.or_optimizer_step.argtypes = [C.c_int, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                          C.POINTER(Cfg), C.POINTER(StepState)]
        lib.or_optimizer_step_ex.argtypes = [C.c_int, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                             C.POINTER(Cfg), C.POINTER(StepState), C.c_int]
        lib.or_bf16_to_float.restype = C.c_float
        lib.or_bf16_to_float.argtypes = [C.c_uint16]
        lib.or_bf16_to_float_n.argtypes = [vp, vp, u64]
        lib.or_unpruned_count.restype = u64
        lib.or_unpruned_count.argtypes = [C.c_double, u64]
        lib.or_magnitude_prune.argtypes = [vp, vp, vp, C.c_int, C.c_double, C.c_int, vp, vp]
        lib.or_synth_f32.argtypes = [vp, u64, u64, u64, u64, C.c_float]
        lib.or_synth_f16.argtypes = [vp, u64, u64, u64, u64, C.c_float, C.c_float]
        lib.or_mt64_seed.argtypes = [C.POINTER(MT64), u64]
        lib.or_mt64_next.restype = u64
        lib.or_mt64_next.argtypes = [C.POINTER(MT64)]
        lib.or_mt64_uniform.argtypes = [C.POINTER(MT64), vp, u64, C.c_float]
        lib.or_dp_sum.argtypes = [vp, C.c_int, u64, vp, vp]
        lib.or_dw_matmul.argtypes = [vp, vp, u64, u64, u64, vp]

    # half.hpp
    def f2h(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty(x.shape, dtype=np.uint16)
        self.lib.or_f2h(_p(x), _p(out), x.size)
        return out

    def h2f(self, h) -> np.ndarray:
        h = np.ascontiguousarray(h, dtype=np.uint16)
        out = np.empty(h.shape, dtype=np.float32)
        self.lib.or_h2f(_p(h), _p(out), h.size)
        return out

    # store.hpp
    def compress(self, dense: np.ndarray, idx: np.ndarray, ind_dense_len: int | None = None):
        dense = np.ascontiguousarray(dense).reshape(-1)
        idx = np.ascontiguousarray(idx, dtype=np.uint32)
        out = np.empty(idx.size, dtype=dense.dtype)
        fn = {2: self.lib.or_compress_u16, 4: self.lib.or_compress_u32}[dense.itemsize]
        rc = fn(_p(dense), dense.size, _p(idx), idx.size,
                dense.size if ind_dense_len is None else ind_dense_len, _p(out))
        if rc:
            raise ValueError("DimensionError")
        return out

    def expand(self, values: np.ndarray, idx: np.ndarray, shape, ind_dense_len=None):
        values = np.ascontiguousarray(values)
        idx = np.ascontiguousarray(idx, dtype=np.uint32)
        numel = int(np.prod(shape))
        out = np.empty(numel, dtype=values.dtype)
        fn = {2: self.lib.or_expand_u16, 4: self.lib.or_expand_u32}[values.itemsize]
        rc = fn(_p(values), values.size, _p(idx), idx.size,
                numel if ind_dense_len is None else ind_dense_len, numel, _p(out))
        if rc:
            raise ValueError("DimensionError")
        return out.reshape(shape)

    # train.hpp
    def adam_update(self, theta, m, v, g, cfg: Cfg, bias1: float, bias2: float) -> None:
        for a in (theta, m, v, g):
            assert a.dtype == np.float32 and a.flags.c_contiguous
        self.lib.or_adam_update(_p(theta), _p(m), _p(v), _p(g), theta.size, C.byref(cfg),
                                C.c_float(bias1), C.c_float(bias2))

    def optimizer_step(self, dense_len, nnz, idx_arena, dense_grads, theta, m, v, g32, theta16,
                       cfg: Cfg, st: StepState, grad_bf16: bool = False) -> bool:
        """dense_grads: uint16 bit patterns, binary16 (the reference) or, with
        grad_bf16, bfloat16."""
        dl = np.ascontiguousarray(dense_len, dtype=np.uint64)
        nz = np.ascontiguousarray(nnz, dtype=np.uint64)
        gp = _ptr_array(dense_grads)
        tp = _ptr_array(theta16)
        return bool(self.lib.or_optimizer_step_ex(len(dl), _p(dl), _p(nz), _p(idx_arena), gp,
                                                  _p(theta), _p(m), _p(v), _p(g32), tp,
                                                  C.byref(cfg), C.byref(st), 1 if grad_bf16 else 0))

    def bf16_to_float(self, h) -> np.ndarray:
        h = np.ascontiguousarray(h, dtype=np.uint16)
        out = np.empty(h.shape, dtype=np.float32)
        self.lib.or_bf16_to_float_n(_p(h), _p(out), h.size)
        return out

    # prune.hpp
    def unpruned_count(self, p: float, n: int) -> int:
        return int(self.lib.or_unpruned_count(p, n))

    def magnitude_prune(self, values, prunable, p: float, scope: int = 0):
        vals = [np.ascontiguousarray(v, dtype=np.float32).reshape(-1) for v in values]
        lens = np.array([v.size for v in vals], dtype=np.uint64)
        pr = np.array([1 if x else 0 for x in prunable], dtype=np.uint8)
        outs = [np.empty(max(1, v.size), dtype=np.uint32) for v in vals]
        counts = np.zeros(len(vals), dtype=np.uint64)
        rc = self.lib.or_magnitude_prune(_ptr_array(vals), _p(lens), _p(pr), len(vals), p, scope,
                                         _ptr_array(outs), _p(counts))
        if rc:
            raise ValueError("ParameterError")
        return [o[: int(c)].copy() for o, c in zip(outs, counts)]

    # synthetic data mirrors
    def synth_f32(self, first: int, n: int, seed: int, sid: int, bound: float) -> np.ndarray:
        out = np.empty(n, dtype=np.float32)
        self.lib.or_synth_f32(_p(out), first, n, seed, sid, C.c_float(bound))
        return out

    def synth_f16(self, first: int, n: int, seed: int, sid: int, bound: float, scale: float):
        out = np.empty(n, dtype=np.uint16)
        self.lib.or_synth_f16(_p(out), first, n, seed, sid, C.c_float(bound), C.c_float(scale))
        return out

    def mt64_uniform(self, seed: int, n: int, bound: float) -> np.ndarray:
        st = MT64()
        self.lib.or_mt64_seed(C.byref(st), seed)
        out = np.empty(n, dtype=np.float32)
        self.lib.or_mt64_uniform(C.byref(st), _p(out), n, C.c_float(bound))
        return out

    def mt64_raw(self, seed: int, n: int) -> np.ndarray:
        st = MT64()
        self.lib.or_mt64_seed(C.byref(st), seed)
        return np.array([self.lib.or_mt64_next(C.byref(st)) for _ in range(n)], dtype=np.uint64)

    def dp_sum(self, bufs):
        bufs = [np.ascontiguousarray(b, dtype=np.float32) for b in bufs]
        n = bufs[0].size
        out = np.empty(n, dtype=np.float32)
        a = np.empty(n, dtype=np.float64)
        self.lib.or_dp_sum(_ptr_array(bufs), len(bufs), n, _p(out), _p(a))
        return out, a

    def dw_matmul(self, x: np.ndarray, dy: np.ndarray) -> np.ndarray:
        """binary16 bits of matmul(transpose(x), dy) (tensor.hpp:88-105)."""
        x = np.ascontiguousarray(x, dtype=np.uint16)
        dy = np.ascontiguousarray(dy, dtype=np.uint16)
        out = np.empty((x.shape[1], dy.shape[1]), dtype=np.uint16)
        self.lib.or_dw_matmul(_p(x), _p(dy), x.shape[0], x.shape[1], dy.shape[1], _p(out))
        return out


class RefLib:
    """The reference itself (unmodified headers) behind extern "C"."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (needs /root/reference at build time)")
        lib = C.CDLL(str(path))
        self.lib = lib
        for n in ("ref_f2h", "ref_h2f"):
            getattr(lib, n).argtypes = [vp, vp, u64]
        lib.ref_compress_u16.argtypes = [vp, u64, vp, u64, u64, vp]
        lib.ref_compress_f32.argtypes = [vp, u64, vp, u64, u64, vp]
        lib.ref_expand_u16.argtypes = [vp, u64, vp, u64, u64, u64, vp]
        lib.ref_expand_f32.argtypes = [vp, u64, vp, u64, u64, u64, vp]
        lib.ref_adam_update.argtypes = [vp, vp, vp, vp, u64, C.POINTER(Cfg), C.c_float, C.c_float]
        lib.ref_config_validate.argtypes = [C.POINTER(Cfg)]
        lib.ref_unpruned_count.restype = u64
        lib.ref_unpruned_count.argtypes = [C.c_double, u64]
        lib.ref_magnitude_prune.argtypes = [vp, vp, vp, C.c_int, C.c_double, C.c_int, vp, vp]
        lib.ref_uniform_symmetric.argtypes = [u64, C.c_float, vp, u64]
        lib.ref_session_create.restype = vp
        lib.ref_session_create.argtypes = [C.c_int, vp, vp, vp, vp, C.POINTER(Cfg)]
        lib.ref_session_destroy.argtypes = [vp]
        lib.ref_session_step.argtypes = [vp, vp]
        lib.ref_session_wrap_grads.restype = vp
        lib.ref_session_wrap_grads.argtypes = [vp, vp]
        lib.ref_grads_destroy.argtypes = [vp]
        lib.ref_session_step_wrapped.argtypes = [vp, vp]
        lib.ref_session_read.argtypes = [vp, C.c_int, vp, vp, vp, vp, vp]
        lib.ref_session_counters.argtypes = [vp, C.POINTER(u64), C.POINTER(C.c_float)]
        lib.ref_session_check_invariants.argtypes = [vp]
        lib.ref_session_measured_bytes.restype = u64
        lib.ref_session_measured_bytes.argtypes = [vp, C.c_int]
        lib.ref_dw_matmul.argtypes = [vp, vp, u64, u64, u64, vp]
        self.has_json = hasattr(lib, "ref_checkpoint_json_roundtrip")  # built with nlohmann/json
        if self.has_json:
            for n in ("ref_checkpoint_json_roundtrip", "ref_index_sets_json_roundtrip"):
                getattr(lib, n).argtypes = [C.c_char_p, C.c_char_p, u64, C.POINTER(u64)]

    def _json_roundtrip(self, fn, text: str):
        need = u64(0)
        cap = 2 * len(text) + 4096
        for _ in range(2):
            buf = C.create_string_buffer(cap)
            rc = fn(text.encode(), buf, cap, C.byref(need))
            if rc != 100:
                return rc, buf.value.decode() if rc == 0 else None
            cap = int(need.value)
        return rc, None

    def checkpoint_json_roundtrip(self, text: str):
        """The reference's checkpoint_from_json + checkpoint_to_json + dump on
        `text`: (status, output text)."""
        return self._json_roundtrip(self.lib.ref_checkpoint_json_roundtrip, text)

    def index_sets_json_roundtrip(self, text: str):
        """index_sets_from_json + index_sets_to_json + dump: (status, text)."""
        return self._json_roundtrip(self.lib.ref_index_sets_json_roundtrip, text)

    def f2h(self, x):
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty(x.shape, dtype=np.uint16)
        self.lib.ref_f2h(_p(x), _p(out), x.size)
        return out

    def h2f(self, h):
        h = np.ascontiguousarray(h, dtype=np.uint16)
        out = np.empty(h.shape, dtype=np.float32)
        self.lib.ref_h2f(_p(h), _p(out), h.size)
        return out

    def compress(self, dense, idx, ind_dense_len=None):
        dense = np.ascontiguousarray(dense).reshape(-1)
        idx = np.ascontiguousarray(idx, dtype=np.uint32)
        out = np.empty(idx.size, dtype=dense.dtype)
        fn = self.lib.ref_compress_u16 if dense.itemsize == 2 else self.lib.ref_compress_f32
        rc = fn(_p(dense), dense.size, _p(idx), idx.size,
                dense.size if ind_dense_len is None else ind_dense_len, _p(out))
        return rc, out

    def expand(self, values, idx, numel, ind_dense_len=None):
        values = np.ascontiguousarray(values)
        idx = np.ascontiguousarray(idx, dtype=np.uint32)
        out = np.empty(numel, dtype=values.dtype)
        fn = self.lib.ref_expand_u16 if values.itemsize == 2 else self.lib.ref_expand_f32
        rc = fn(_p(values), values.size, _p(idx), idx.size,
                numel if ind_dense_len is None else ind_dense_len, numel, _p(out))
        return rc, out

    def dw_matmul(self, x, dy):
        x = np.ascontiguousarray(x, dtype=np.uint16)
        dy = np.ascontiguousarray(dy, dtype=np.uint16)
        out = np.empty((x.shape[1], dy.shape[1]), dtype=np.uint16)
        rc = self.lib.ref_dw_matmul(_p(x), _p(dy), x.shape[0], x.shape[1], dy.shape[1], _p(out))
        return rc, out

    def adam_update(self, theta, m, v, g, cfg: Cfg, bias1, bias2):
        self.lib.ref_adam_update(_p(theta), _p(m), _p(v), _p(g), theta.size, C.byref(cfg),
                                 C.c_float(bias1), C.c_float(bias2))

    def unpruned_count(self, p, n):
        return int(self.lib.ref_unpruned_count(p, n))

    def magnitude_prune(self, values, prunable, p, scope=0):
        vals = [np.ascontiguousarray(v, dtype=np.float32).reshape(-1) for v in values]
        lens = np.array([v.size for v in vals], dtype=np.uint64)
        pr = np.array([1 if x else 0 for x in prunable], dtype=np.uint8)
        outs = [np.empty(max(1, v.size), dtype=np.uint32) for v in vals]
        counts = np.zeros(len(vals), dtype=np.uint64)
        rc = self.lib.ref_magnitude_prune(_ptr_array(vals), _p(lens), _p(pr), len(vals), p, scope,
                                          _ptr_array(outs), _p(counts))
        return rc, [o[: int(c)].copy() for o, c in zip(outs, counts)]

    def uniform_symmetric(self, seed, bound, n):
        out = np.empty(n, dtype=np.float32)
        self.lib.ref_uniform_symmetric(seed, C.c_float(bound), _p(out), n)
        return out


class RefSession:
    """SamoTrainer::optimizer_step of the unmodified reference, at any scale."""

    def __init__(self, ref: RefLib, dense_len, idx_sets, theta32_sets, cfg: Cfg):
        self.ref = ref
        self.dense_len = np.ascontiguousarray(dense_len, dtype=np.uint64)
        self.nnz = np.array([len(i) for i in idx_sets], dtype=np.uint64)
        self._idx = [np.ascontiguousarray(i, dtype=np.uint32) for i in idx_sets]
        self._th = [np.ascontiguousarray(t, dtype=np.float32) for t in theta32_sets]
        self.h = ref.lib.ref_session_create(len(self.dense_len), _p(self.dense_len), _p(self.nnz),
                                            _ptr_array(self._idx), _ptr_array(self._th),
                                            C.byref(cfg))
        self._wrapped = None

    def step(self, dense_grads) -> bool:
        g = [np.ascontiguousarray(x, dtype=np.uint16) for x in dense_grads]
        return bool(self.ref.lib.ref_session_step(self.h, _ptr_array(g)))

    def wrap(self, dense_grads) -> None:
        g = [np.ascontiguousarray(x, dtype=np.uint16) for x in dense_grads]
        if self._wrapped:
            self.ref.lib.ref_grads_destroy(self._wrapped)
        self._wrapped = self.ref.lib.ref_session_wrap_grads(self.h, _ptr_array(g))

    def step_wrapped(self) -> bool:
        return bool(self.ref.lib.ref_session_step_wrapped(self.h, self._wrapped))

    def read(self, layer: int):
        n = int(self.nnz[layer])
        d = int(self.dense_len[layer])
        th, m, v, g = (np.empty(n, np.float32) for _ in range(4))
        t16 = np.empty(d, np.uint16)
        self.ref.lib.ref_session_read(self.h, layer, _p(th), _p(m), _p(v), _p(g), _p(t16))
        return {"theta32": th, "adam_m": m, "adam_v": v, "grad32": g, "theta16": t16}

    def counters(self):
        sk = u64()
        gn = C.c_float()
        self.ref.lib.ref_session_counters(self.h, C.byref(sk), C.byref(gn))
        return int(sk.value), float(gn.value)

    def check_invariants(self) -> int:
        return int(self.ref.lib.ref_session_check_invariants(self.h))

    def close(self):
        if self._wrapped:
            self.ref.lib.ref_grads_destroy(self._wrapped)
            self._wrapped = None
        if self.h:
            self.ref.lib.ref_session_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
