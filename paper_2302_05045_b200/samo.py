"""Python mirror of the reference operator interface for the SAMO step path.

Same names, argument meaning and error behaviour as the reference's C++ API
(/root/reference/proj/include/samo): `compress`, `expand`, `adam_update`,
`magnitude_prune`, `unpruned_count`, `make_layer_state`-style model init and a
`SamoTrainer`-style step driver — over CUDA tensors, every call going through
the C ABI of libsamo_cuda.so (include/samo_cuda.h).  torch is used only for
device memory and streams.

binary16 data is carried in torch.float16 / torch.int16 tensors and handled as
raw 16-bit patterns (the reference's `Half` is a storage type, half.hpp:75-103);
fp32 data in torch.float32; index sets in torch.int32 holding uint32 values.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np
import torch

from . import _abi
from ._abi import (DimensionError, ParameterError, SamoIndexError, StateError,  # noqa: F401
                   ConfigError, CudaError, NcclError, OptimizerConfig, StepRecord)

PER_LAYER = 0   # PruneScope::per_layer (prune.hpp:61)
GLOBAL = 1      # PruneScope::global


def _vp(t: torch.Tensor | None) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


def _stream(stream: torch.cuda.Stream | None = None) -> C.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _require_cuda(*ts: torch.Tensor) -> None:
    for t in ts:
        if t is not None and (not t.is_cuda or not t.is_contiguous()):
            raise ParameterError("expected contiguous CUDA tensors (the SAMO path has no CPU fallback)")


def _bits16(t: torch.Tensor) -> torch.Tensor:
    if t.element_size() != 2:
        raise ParameterError("expected a 16-bit tensor")
    return t


# ---------------------------------------------------------------------------
# half.hpp


def float_to_half_bits(x: torch.Tensor) -> torch.Tensor:
    """Half(float) for every element (half.hpp:13-49); returns int16 bit patterns."""
    _require_cuda(x)
    out = torch.empty(x.shape, dtype=torch.int16, device=x.device)
    _abi.call("samo_float_to_half", _vp(x), _vp(out), x.numel(), _stream())
    return out


def half_bits_to_float(h: torch.Tensor) -> torch.Tensor:
    """float(Half) for every element (half.hpp:52-71)."""
    _require_cuda(h)
    _bits16(h)
    out = torch.empty(h.shape, dtype=torch.float32, device=h.device)
    _abi.call("samo_half_to_float", _vp(h), _vp(out), h.numel(), _stream())
    return out


# ---------------------------------------------------------------------------
# prune.hpp


@dataclass
class PrunedIndexSet:
    """prune.hpp:21-27: strictly ascending uint32 linear indices (< dense_len)."""
    layer_id: str
    dense_len: int
    indices: torch.Tensor  # int32 CUDA tensor carrying uint32 values

    def count(self) -> int:
        return int(self.indices.numel())

    def as_int64(self) -> torch.Tensor:
        """The indices widened for torch indexing: values >= 2^31 (layers up to
        2^32 - 1 elements, prune.hpp:106-109) are held as negative int32, so a
        plain .long() would sign-extend them."""
        return self.indices.long() & 0xFFFFFFFF


@dataclass
class LayerParams:
    """prune.hpp:65-69."""
    layer_id: str
    values: torch.Tensor  # fp32 CUDA tensor, any shape
    prunable: bool = True


def index_sets_to_json(sets: Sequence[PrunedIndexSet]) -> str:
    """index_sets_to_json(sets).dump() (serialize.hpp:84-93)."""
    from . import checkpoint_json as cj
    return cj.index_sets_dumps(sets)


def index_sets_from_json(text: str, device: str = "cuda") -> list[PrunedIndexSet]:
    """index_sets_from_json (serialize.hpp:95-119), validated as the
    reference does (ConfigError); indices land on `device`."""
    from . import checkpoint_json as cj
    return [PrunedIndexSet(lid, n, torch.from_numpy(idx.view(np.int32).copy()).to(device))
            for lid, n, idx in cj.index_sets_loads(text)]


def unpruned_count(p: float, n: int) -> int:
    """detail::unpruned_count (prune.hpp:76-79)."""
    return int(_abi.load().samo_unpruned_count(float(p), int(n)))


def magnitude_prune(layers: Sequence[LayerParams], p: float,
                    scope: int = PER_LAYER) -> list[PrunedIndexSet]:
    """magnitude_prune (prune.hpp:99-170), on the device (kernel K0)."""
    n = len(layers)
    for lp in layers:
        _require_cuda(lp.values)
        if lp.values.dtype != torch.float32:
            raise ParameterError("magnitude_prune expects fp32 values")
    outs = [torch.empty(max(1, lp.values.numel()), dtype=torch.int32, device=lp.values.device)
            for lp in layers]
    vals = (C.c_void_p * max(1, n))(*[lp.values.data_ptr() for lp in layers])
    lens = (C.c_uint64 * max(1, n))(*[lp.values.numel() for lp in layers])
    prun = (C.c_uint8 * max(1, n))(*[1 if lp.prunable else 0 for lp in layers])
    optr = (C.c_void_p * max(1, n))(*[o.data_ptr() for o in outs])
    counts = (C.c_uint64 * max(1, n))()
    _abi.call("samo_magnitude_prune", vals, lens, prun, n, float(p), int(scope), optr, counts,
              _stream())
    return [PrunedIndexSet(lp.layer_id, lp.values.numel(), outs[i][: counts[i]].clone())
            for i, lp in enumerate(layers)]


# ---------------------------------------------------------------------------
# store.hpp


def compress(dense: torch.Tensor, ind: PrunedIndexSet) -> torch.Tensor:
    """compress<T> (store.hpp:58-69): out[k] = dense.flat[ind.indices[k]]."""
    _require_cuda(dense, ind.indices)
    out = torch.empty(ind.count(), dtype=dense.dtype, device=dense.device)
    name = {2: "samo_compress_u16", 4: "samo_compress_u32"}.get(dense.element_size())
    if name is None:
        raise ParameterError("compress supports 16- and 32-bit elements")
    _abi.call(name, _vp(dense), dense.numel(), _vp(ind.indices), ind.count(), ind.dense_len,
              _vp(out), _stream())
    return out


def dw_gemm(x: torch.Tensor, dy: torch.Tensor) -> torch.Tensor:
    """Dense weight gradient x^T . dy as binary16 (tcgen05, fp32 accumulate):
    matmul(transpose(x), dy) of tensor.hpp:88-105 up to summation order."""
    _require_cuda(x, dy)
    if x.dim() != 2 or dy.dim() != 2 or x.shape[0] != dy.shape[0]:
        raise DimensionError("dw_gemm expects x [batch, in] and dy [batch, out]")
    x, dy = _bits16(x).contiguous(), _bits16(dy).contiguous()
    out = torch.empty((x.shape[1], dy.shape[1]), dtype=x.dtype, device=x.device)
    _abi.call("samo_dw_gemm_f16", _vp(x), _vp(dy), x.shape[0], x.shape[1], dy.shape[1], _vp(out), _stream())
    return out


def expand(values: torch.Tensor, ind: PrunedIndexSet, shape: Sequence[int]) -> torch.Tensor:
    """expand<T> (store.hpp:72-87): zeros except out.flat[ind.indices[k]] = values[k]."""
    _require_cuda(values, ind.indices)
    numel = 1
    for e in shape:
        if int(e) <= 0:
            raise DimensionError("tensor extents must be positive")
        numel *= int(e)
    out = torch.empty(tuple(int(e) for e in shape), dtype=values.dtype, device=values.device)
    name = {2: "samo_expand_u16", 4: "samo_expand_u32"}.get(values.element_size())
    if name is None:
        raise ParameterError("expand supports 16- and 32-bit elements")
    _abi.call(name, _vp(values), values.numel(), _vp(ind.indices), ind.count(), ind.dense_len,
              numel, _vp(out), _stream())
    return out


def downcast_expand(theta32: torch.Tensor, ind: PrunedIndexSet,
                    shape: Sequence[int]) -> torch.Tensor:
    """expand<Half>(Half(theta32), ind, shape) (train.hpp:647-651) in one pass."""
    _require_cuda(theta32, ind.indices)
    numel = 1
    for e in shape:
        numel *= int(e)
    if numel != ind.dense_len:
        raise DimensionError("expand: shape does not match index set dense length")
    if theta32.numel() != ind.count():
        raise DimensionError("expand: value count does not match index set")
    out = torch.empty(tuple(int(e) for e in shape), dtype=torch.float16, device=theta32.device)
    _abi.call("samo_downcast_expand", _vp(theta32), ind.count(), _vp(ind.indices), ind.dense_len,
              _vp(out), _stream())
    return out


# ---------------------------------------------------------------------------
# train.hpp


def validate(cfg: OptimizerConfig) -> None:
    """OptimizerConfig::validate (train.hpp:78-86)."""
    _abi.call("samo_optimizer_config_validate", C.byref(cfg))


def adam_update(theta: torch.Tensor, m: torch.Tensor, v: torch.Tensor, g: torch.Tensor,
                cfg: OptimizerConfig, bias1: float, bias2: float) -> None:
    """adam_update (train.hpp:332-347), in place on device spans."""
    _require_cuda(theta, m, v, g)
    n = theta.numel()
    if not (m.numel() == v.numel() == g.numel() == n):
        raise DimensionError("adam_update: span lengths differ")
    _abi.call("samo_adam_update", _vp(theta), _vp(m), _vp(v), _vp(g), n, C.byref(cfg),
              C.c_float(bias1), C.c_float(bias2), _stream())


# ---------------------------------------------------------------------------
# Gradient exchange communicator


class Communicator:
    """NCCL communicator for the compressed-gradient exchange (one per rank)."""

    def __init__(self, unique_id: bytes, nranks: int, rank: int):
        if len(unique_id) != 128:
            raise ParameterError("unique id must be 128 bytes")
        buf = (C.c_uint8 * 128)(*unique_id)
        h = C.c_void_p()
        _abi.call("samo_comm_create", buf, int(nranks), int(rank), C.byref(h))
        self._h = h
        self.nranks = int(nranks)
        self.rank = int(rank)

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _abi.call("samo_comm_unique_id", buf)
        return bytes(buf)

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def allreduce_sum_(self, t: torch.Tensor) -> torch.Tensor:
        _require_cuda(t)
        if t.dtype != torch.float32:
            raise ParameterError("allreduce expects fp32")
        _abi.call("samo_allreduce_sum_f32", self._h, _vp(t), t.numel(), _stream())
        return t

    def close(self) -> None:
        if self._h:
            _abi.load().samo_comm_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# Model state + step driver (store.hpp:22-55, 150-197; train.hpp:574-704)


@dataclass
class LayerSpec:
    layer_id: str
    shape: tuple[int, ...]
    nnz: int

    @property
    def dense_len(self) -> int:
        n = 1
        for e in self.shape:
            n *= int(e)
        return n


class SamoModel:
    """Device-resident compressed model state with the fused step driver.

    Mirrors ModelState (store.hpp:42-55) + SamoTrainer::optimizer_step
    (train.hpp:617-656): flat arenas for theta32/m/v/grad32/indices, a dense
    binary16 theta16 per layer, device-resident Adam scalars.  The step is
    K1 gather+unscale -> NCCL exchange (when a communicator is attached) -> K23
    Adam+downcast+expand, with no host synchronisation.
    """

    def __init__(self, layers: Sequence[LayerSpec], tile_elems: int = 0):
        self.layers = list(layers)
        descs = (_abi.LayerDesc * max(1, len(self.layers)))(
            *[_abi.LayerDesc(l.dense_len, l.nnz) for l in self.layers])
        h = C.c_void_p()
        _abi.call("samo_model_create", descs, len(self.layers), int(tile_elems), C.byref(h))
        self._h = h
        self._grads_keepalive: list[torch.Tensor] = []
        self._sink_keepalive: list[torch.Tensor] = []

    # -- construction ------------------------------------------------------
    @classmethod
    def from_index_sets(cls, sets: Sequence[PrunedIndexSet], shapes: Sequence[Sequence[int]],
                        tile_elems: int = 0) -> "SamoModel":
        specs = [LayerSpec(s.layer_id, tuple(int(e) for e in shp), s.count())
                 for s, shp in zip(sets, shapes)]
        model = cls(specs, tile_elems)
        for l, s in enumerate(sets):
            model.set_indices(l, s.indices)
        model.finalize()
        return model

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def close(self) -> None:
        if self._h:
            _abi.load().samo_model_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def set_indices(self, layer: int, idx: torch.Tensor) -> None:
        on_host = not idx.is_cuda
        idx = idx.contiguous()
        _abi.call("samo_model_set_indices", self._h, int(layer), _vp(idx), idx.numel(),
                  1 if on_host else 0, _stream())

    def finalize(self) -> None:
        _abi.call("samo_model_finalize", self._h, _stream())

    def init_layer(self, layer: int, dense_init: torch.Tensor) -> None:
        """make_layer_state (store.hpp:150-168) from dense fp32 initial values."""
        _require_cuda(dense_init)
        if dense_init.dtype != torch.float32:
            raise ParameterError("init values must be fp32")
        _abi.call("samo_model_init_layer", self._h, int(layer), _vp(dense_init),
                  dense_init.numel(), _stream())

    def set_config(self, cfg: OptimizerConfig) -> None:
        _abi.call("samo_model_set_config", self._h, C.byref(cfg))

    GRAD_F16, GRAD_BF16 = 0, 1

    def set_grad_dtype(self, dtype) -> None:
        """Element type of the dense gradients: torch.float16 (binary16, the
        reference's Half; default) or torch.bfloat16 (widened exactly)."""
        code = {torch.float16: self.GRAD_F16, "f16": self.GRAD_F16, "fp16": self.GRAD_F16,
                torch.bfloat16: self.GRAD_BF16, "bf16": self.GRAD_BF16}.get(dtype)
        if code is None:
            raise ParameterError(f"gradient dtype must be float16 or bfloat16, not {dtype}")
        _abi.call("samo_model_set_grad_dtype", self._h, code)

    @property
    def grad_dtype(self) -> torch.dtype:
        return torch.bfloat16 if _abi.load().samo_model_grad_dtype(self._h) == self.GRAD_BF16 else torch.float16

    def _check_grad(self, g: torch.Tensor) -> None:
        _bits16(g)
        if g.dtype in (torch.float16, torch.bfloat16) and g.dtype != self.grad_dtype:
            raise ParameterError(f"gradient is {g.dtype}, the model expects {self.grad_dtype} (set_grad_dtype)")

    def attach_comm(self, comm: Communicator | None) -> None:
        _abi.call("samo_model_attach_comm", self._h, comm.handle if comm else C.c_void_p())

    EXCHANGE_NONE, EXCHANGE_ALLREDUCE, EXCHANGE_SHARDED, EXCHANGE_P2P = 0, 1, 2, 3

    @staticmethod
    def attach_local_group(models: Sequence["SamoModel"]) -> None:
        """Test harness (samo_model_attach_local_group): the models, all on the
        current device, become the ranks of one peer-to-peer group with no
        NCCL; step them together with local_group_step."""
        hs = (C.c_void_p * len(models))(*[m._h.value for m in models])
        _abi.call("samo_model_attach_local_group", hs, len(models))

    @staticmethod
    def local_group_step(models: Sequence["SamoModel"]) -> None:
        """One pipelined peer-to-peer step of every rank of a local group,
        phase by phase on the current stream (samo_local_group_step)."""
        hs = (C.c_void_p * len(models))(*[m._h.value for m in models])
        _abi.call("samo_local_group_step", hs, len(models), _stream())

    @staticmethod
    def local_group_step_sunk(models: Sequence["SamoModel"]) -> None:
        """Test harness: the group's step after every member's backward sinks
        (samo_local_group_step_sunk)."""
        hs = (C.c_void_p * len(models))(*[m._h.value for m in models])
        _abi.call("samo_local_group_step_sunk", hs, len(models), _stream())

    def set_exchange(self, mode: int) -> None:
        """EXCHANGE_ALLREDUCE (replicated state), EXCHANGE_SHARDED (ZeRO-1 on
        the compressed state, NCCL reduce-scatter / all-gather) or EXCHANGE_P2P
        (ZeRO-1 with the exchange fused into the shard kernel over NVLink peer
        memory); -1 restores the default."""
        _abi.call("samo_model_set_exchange", self._h, int(mode))

    def exchange_mode(self) -> int:
        return int(_abi.load().samo_model_exchange_mode(self._h))

    def shard_ranges(self) -> list[tuple[int, int]]:
        """Compressed-arena ranges [k0, k1) this rank updates (all of them
        unless the exchange is sharded)."""
        c, st, nb, rk = C.c_uint64(), C.c_uint64(), C.c_int(), C.c_int()
        _abi.call("samo_model_shard_layout", self._h, C.byref(c), C.byref(st), C.byref(nb),
                  C.byref(rk))
        n = self.totals()[1]
        out = []
        for b in range(nb.value):
            k0 = min(b * st.value + rk.value * c.value, n)
            k1 = min(b * st.value + (rk.value + 1) * c.value, n)
            if k1 > k0:
                out.append((k0, k1))
        return out

    # -- step ----------------------------------------------------------------
    def set_grads(self, grads: Sequence[torch.Tensor]) -> None:
        """Dense 16-bit gradients of the step (the backward sink's input):
        binary16, or bfloat16 after set_grad_dtype(torch.bfloat16); int16
        tensors pass raw bit patterns of the model's type."""
        if len(grads) != len(self.layers):
            raise DimensionError("one dense gradient per layer required")
        for g, l in zip(grads, self.layers):
            _require_cuda(g)
            self._check_grad(g)
            if g.numel() != l.dense_len:
                raise DimensionError(f"{l.layer_id}: gradient length does not match layer")
        ptrs = (C.c_void_p * max(1, len(grads)))(*[g.data_ptr() for g in grads])
        _abi.call("samo_model_set_grads", self._h, ptrs, _stream())
        self._grads_keepalive = list(grads)

    def gather(self) -> None:
        _abi.call("samo_model_gather", self._h, _stream())

    def sink_dense(self, layer: int, grad: torch.Tensor) -> None:
        """Backward sink (train.hpp:596-611) of one layer's dense binary16
        gradient: K1 on that layer only.  Single-GPU models."""
        _require_cuda(grad)
        self._check_grad(grad)
        if grad.numel() != self.layers[layer].dense_len:
            raise DimensionError(f"{self.layers[layer].layer_id}: gradient length does not match layer")
        _abi.call("samo_model_sink_dense", self._h, layer, _vp(grad), _stream())
        self._sink_keepalive.append(grad)

    def sink_dw(self, layer: int, x: torch.Tensor, dy: torch.Tensor) -> None:
        """Fused backward sink: dW = x^T . dy (mlp_backward, train.hpp:304-305)
        on the tensor cores with the gather in the GEMM epilogue; x [batch, in],
        dy [batch, out] binary16."""
        _require_cuda(x, dy)
        if x.dim() != 2 or dy.dim() != 2 or x.shape[0] != dy.shape[0]:
            raise DimensionError("sink_dw expects x [batch, in] and dy [batch, out]")
        x, dy = _bits16(x).contiguous(), _bits16(dy).contiguous()
        _abi.call("samo_model_sink_dw", self._h, layer, _vp(x), _vp(dy), x.shape[0], x.shape[1],
                  dy.shape[1], _stream())
        self._sink_keepalive.extend((x, dy))

    def exchange(self) -> None:
        _abi.call("samo_model_exchange", self._h, _stream())

    def p2p_features(self) -> dict:
        """Peer-to-peer mechanisms in use: mapped, push (K1 pushes the gradients to their owners)."""
        f = int(_abi.load().samo_model_p2p_features(self._h))
        return {"mapped": bool(f & 1), "push": bool(f & 2)}

    def step_sunk(self) -> None:
        """The step after the backward sinks: exchange (peer-to-peer) + update."""
        _abi.call("samo_model_step_sunk", self._h, _stream())
        self._sink_keepalive = []

    def update(self) -> None:
        _abi.call("samo_model_update", self._h, _stream())
        self._sink_keepalive = []  # stream-ordered: later allocations reuse safely

    def step(self, graph: bool = False) -> None:
        """gather + exchange + Adam/downcast/expand; device-resident, async."""
        _abi.call("samo_model_step_graph" if graph else "samo_model_step", self._h, _stream())

    def step_record(self) -> StepRecord:
        rec = StepRecord()
        _abi.call("samo_model_step_record", self._h, C.byref(rec), _stream())
        return rec

    def set_step_record(self, rec: StepRecord) -> None:
        _abi.call("samo_model_set_step_record", self._h, C.byref(rec), _stream())

    def check_invariants(self) -> None:
        """check_state_invariants (store.hpp:171-197) -> StateError."""
        _abi.call("samo_model_check_invariants", self._h, _stream())

    # -- views -----------------------------------------------------------------
    def view(self, layer: int) -> _abi.LayerView:
        v = _abi.LayerView()
        _abi.call("samo_model_layer_view", self._h, int(layer), C.byref(v))
        return v

    def totals(self) -> tuple[int, int, int]:
        phi, nnz, nt = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _abi.call("samo_model_totals", self._h, C.byref(phi), C.byref(nnz), C.byref(nt))
        return phi.value, nnz.value, nt.value

    def device_bytes(self) -> int:
        return int(_abi.load().samo_model_device_bytes(self._h))

    def memory(self) -> dict:
        """Device footprint beside the reference's measured_bytes (store.hpp:129-147)."""
        r = _abi.MemoryReport()
        _abi.call("samo_model_memory", self._h, C.byref(r))
        return {k: int(getattr(r, k)) for k, _ in r._fields_}

    def save(self, path: str) -> None:
        """Binary checkpoint: indices, theta32, adam_m, adam_v per layer + Adam
        scalars (the fields of serialize.hpp:120-190)."""
        _abi.call("samo_model_save", self._h, str(path).encode(), _stream())

    @classmethod
    def load(cls, path: str, layers: Sequence[LayerSpec] | None = None,
             tile_elems: int = 0) -> "SamoModel":
        """Rebuilds a model from samo_model_save output; theta16 is rebuilt by
        downcast+expand (serialize.hpp:184-186)."""
        h = C.c_void_p()
        _abi.call("samo_model_load", str(path).encode(), int(tile_elems), C.byref(h), _stream())
        model = cls.__new__(cls)
        model._h = h
        model._grads_keepalive = []
        model._sink_keepalive = []
        n = int(_abi.load().samo_model_num_layers(h))
        if layers is None:
            layers = []
            for l in range(n):
                v = _abi.LayerView()
                _abi.call("samo_model_layer_view", h, l, C.byref(v))
                layers.append(LayerSpec(f"l{l}", (int(v.dense_len),), int(v.nnz)))
        model.layers = list(layers)
        return model

    def to_checkpoint_json(self) -> str:
        """checkpoint_to_json(state).dump() (serialize.hpp:124-135): per layer
        its id, shape, indices, theta32, adam_m, adam_v.  For small models —
        the binary save() carries the same fields at any scale.  Refused, as
        save() refuses it, when the state is sharded across ranks (theta32 /
        m / v are then only authoritative on this rank's shard)."""
        from . import checkpoint_json as cj
        if self.exchange_mode() in (self.EXCHANGE_SHARDED, self.EXCHANGE_P2P):
            raise StateError("sharded state: theta32/m/v are only authoritative on each rank's shard")
        layers = []
        for l, spec in enumerate(self.layers):
            idx = self.read(l, "indices").cpu().numpy().view(np.uint32)
            layers.append(cj.CheckpointLayer(spec.layer_id, tuple(spec.shape), idx,
                                             *(self.read(l, k).cpu().numpy() for k in ("theta32", "adam_m", "adam_v"))))
        return cj.dumps(layers)

    @classmethod
    def from_checkpoint_json(cls, text: str, tile_elems: int = 0) -> "SamoModel":
        """checkpoint_from_json (serialize.hpp:137-190), validated as the
        reference does (ConfigError), theta16 rebuilt by downcast + expand.
        The JSON has no Adam scalars, so the step counter and beta powers start
        afresh, as a SamoTrainer built on the loaded state does.  Goes through
        the binary loader (samo_model_load)."""
        import os
        import struct
        import tempfile
        from . import checkpoint_json as cj
        layers = cj.loads(text)
        head = struct.pack("<8sIIII", b"SAMOCKPT", 1, len(layers), int(tile_elems) or 16384, 0)
        head += struct.pack("<QQfffI", 0, 0, 1.0, 1.0, 0.0, 0)  # samo_step_record: a fresh trainer
        body = b"".join(struct.pack("<QQ", int(np.prod(l.shape)), l.indices.size) for l in layers)
        fd, path = tempfile.mkstemp(suffix=".samockpt")
        try:
            with os.fdopen(fd, "wb") as f:
                f.write(head + body)
                for k in ("indices", "theta32", "adam_m", "adam_v"):
                    for l in layers:
                        f.write(np.ascontiguousarray(getattr(l, k)).tobytes())
            specs = [LayerSpec(l.layer_id, tuple(l.shape), int(l.indices.size)) for l in layers]
            return cls.load(path, layers=specs, tile_elems=tile_elems)
        finally:
            os.unlink(path)

    _FIELDS = {"theta16": (torch.float16, "dense"), "theta32": (torch.float32, "nnz"),
               "adam_m": (torch.float32, "nnz"), "adam_v": (torch.float32, "nnz"),
               "grad32": (torch.float32, "nnz"), "indices": (torch.int32, "nnz"),
               "grad16": (torch.float16, "nnz")}

    def read(self, layer: int, name: str) -> torch.Tensor:
        """Copy of one per-layer buffer (device tensor)."""
        v = self.view(layer)
        dtype, kind = self._FIELDS[name]
        n = v.dense_len if kind == "dense" else v.nnz
        out = torch.empty(int(n), dtype=dtype, device="cuda")
        if n:
            _abi.call("samo_copy_async", _vp(out), C.c_void_p(getattr(v, name)),
                      int(n) * out.element_size(), _stream())
        return out.view(self.layers[layer].shape) if kind == "dense" else out

    def write(self, layer: int, name: str, src: torch.Tensor) -> None:
        """Overwrite one per-layer buffer (e.g. warm Adam moments on resume)."""
        v = self.view(layer)
        dtype, kind = self._FIELDS[name]
        n = v.dense_len if kind == "dense" else v.nnz
        if src.numel() != n or src.element_size() != torch.empty(0, dtype=dtype).element_size():
            raise DimensionError(f"write {name}: size mismatch")
        src = src.contiguous()
        if n:
            _abi.call("samo_copy_async", C.c_void_p(getattr(v, name)), _vp(src),
                      int(n) * src.element_size(), _stream())


def kernel_launch_count() -> int:
    return int(_abi.load().samo_kernel_launch_count())


def synth_uniform_f32(n: int, seed: int, stream_id: int, bound: float,
                      out: torch.Tensor | None = None) -> torch.Tensor:
    out = out if out is not None else torch.empty(n, dtype=torch.float32, device="cuda")
    _abi.call("samo_synth_uniform_f32", _vp(out), int(n), int(seed), int(stream_id),
              C.c_float(bound), _stream())
    return out


def synth_uniform_f16(n: int, seed: int, stream_id: int, bound: float, scale: float,
                      out: torch.Tensor | None = None) -> torch.Tensor:
    out = out if out is not None else torch.empty(n, dtype=torch.float16, device="cuda")
    _abi.call("samo_synth_uniform_f16", _vp(out), int(n), int(seed), int(stream_id),
              C.c_float(bound), C.c_float(scale), _stream())
    return out
