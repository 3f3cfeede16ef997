"""JSON checkpoints in the reference's schema (serialize.hpp:121-190).

    {"layers": [{"layer_id": str, "shape": [...], "indices": [...],
                 "theta32": [...], "adam_m": [...], "adam_v": [...]}]}

The reference keeps JSON for small models and its tests
(serialize_test.cpp:29-93); at GPT scale the binary checkpoint
(samo_model_save / samo_model_load) carries the same fields.  This module is
host-side format conversion only (numpy arrays in, numpy arrays out); the
model glue is SamoModel.to_checkpoint_json / from_checkpoint_json.

Compatibility with the reference, checked against its own
checkpoint_from_json / checkpoint_to_json in tests/test_checkpoint_json.py:
* values are fp32 widened to double and written with round-trip digits in
  nlohmann's fixed/exponent layout.  Every value parses back to the same fp32
  bits either way.  The texts match byte for byte except where nlohmann's
  Grisu2 picks a different, equally round-tripping, last digit (about 0.7% of
  random fp32 values);
* non-finite values are written as null, as nlohmann writes them, and are
  rejected on load, as the reference rejects them ("bad value");
* integer fields are read as nlohmann's get<uintN_t>() reads them: floats
  truncate, negative integers wrap modulo 2^N (then face the range checks),
  booleans read as 0 / 1;
  only values whose C++ conversion is undefined (non-finite, |x| >= 2^63)
  are rejected where the reference's behaviour is unspecified;
* load rejects exactly what checkpoint_from_json rejects, with ConfigError:
  - a checkpoint that is not an object;
  - unknown keys at either level;
  - a missing key or a value of the wrong type;
  - indices that are not strictly ascending or not below numel(shape);
  - theta32 / adam_m / adam_v lengths that differ from the index count.
  A zero shape extent is a DimensionError, as the reference's Tensor raises.
* Keys are written in sorted order, as nlohmann's std::map stores them.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass
from decimal import Decimal

import numpy as np

from ._abi import ConfigError, DimensionError, ParameterError

LAYER_KEYS = ("layer_id", "shape", "indices", "theta32", "adam_m", "adam_v")


@dataclass
class CheckpointLayer:
    layer_id: str
    shape: tuple[int, ...]
    indices: np.ndarray  # uint32, strictly ascending, < numel(shape)
    theta32: np.ndarray  # float32 [len(indices)]
    adam_m: np.ndarray
    adam_v: np.ndarray


def _number(x: float) -> str:
    """A double in nlohmann::json's layout (format_buffer): fixed notation
    while the decimal point lies within (-4, 15] digits of the shortest
    round-trip digits, else d.ddde+XX; integral values get '.0'; non-finite
    values become null."""
    if not math.isfinite(x):
        return "null"
    if x == 0.0:
        return "-0.0" if math.copysign(1.0, x) < 0 else "0.0"
    t = Decimal(repr(abs(x))).normalize().as_tuple()
    d = "".join(map(str, t.digits))
    k = len(d)
    n = k + t.exponent  # value = 0.d x 10^n
    sign = "-" if x < 0 else ""
    if k <= n <= 15:
        return f"{sign}{d}{'0' * (n - k)}.0"
    if 0 < n <= 15:
        return f"{sign}{d[:n]}.{d[n:]}"
    if -4 < n <= 0:
        return f"{sign}0.{'0' * (-n)}{d}"
    e = n - 1
    mant = d if k == 1 else f"{d[0]}.{d[1:]}"
    return f"{sign}{mant}e{'-' if e < 0 else '+'}{abs(e):02d}"


def _array(a: np.ndarray) -> str:
    return "[" + ",".join(_number(float(x)) for x in np.asarray(a, dtype=np.float32).tolist()) + "]"


def dumps(layers: list[CheckpointLayer]) -> str:
    """checkpoint_to_json(state).dump() (serialize.hpp:124-135): keys sorted as
    nlohmann's std::map holds them, no whitespace."""
    out = []
    for l in layers:
        idx = ",".join(str(int(i)) for i in np.asarray(l.indices, dtype=np.uint32).tolist())
        shape = ",".join(str(int(e)) for e in l.shape)
        out.append(f'{{"adam_m":{_array(l.adam_m)},"adam_v":{_array(l.adam_v)},"indices":[{idx}],'
                   f'"layer_id":{json.dumps(str(l.layer_id), ensure_ascii=False)},"shape":[{shape}],'
                   f'"theta32":{_array(l.theta32)}}}')
    return '{"layers":[' + ",".join(out) + "]}"


def _no_constants(name: str):
    """NaN / Infinity tokens are not JSON (Python's parser accepts them)."""
    raise ConfigError(f"not valid JSON: {name}")


def _required(obj: dict, key: str, where: str):
    if key not in obj:
        raise ConfigError(f"missing key '{key}' in {where}")
    return obj[key]


def _uint(x, key: str, bits: int) -> int:
    """One value as nlohmann's get<uintN_t>() reads it: a JSON integer is
    static_cast (wraps modulo 2^bits, negatives included); a JSON float is
    truncated toward zero, then wraps the same way (what gcc's x86-64
    conversion does for |x| < 2^63); a JSON boolean reads as 0 / 1.  Beyond
    that the C++ cast is undefined behaviour; those values — and
    non-numbers — are rejected (ConfigError)."""
    if isinstance(x, bool):
        return int(x)
    if not isinstance(x, (int, float)):
        raise ConfigError(f"bad value for '{key}' in layer")
    if isinstance(x, int) and -(1 << 63) <= x < (1 << 64):
        return x % (1 << bits)
    x = float(x)  # integers beyond 64 bits parse as floats in nlohmann
    if not math.isfinite(x) or abs(x) >= 2.0**63:
        raise ConfigError(f"bad value for '{key}' in layer")
    return math.trunc(x) % (1 << bits)


def _uints(v, key: str, bits: int) -> list[int]:
    if not isinstance(v, list):
        raise ConfigError(f"bad value for '{key}' in layer")
    return [_uint(x, key, bits) for x in v]


def _f32s(v, key: str) -> np.ndarray:
    if not isinstance(v, list) or not all(isinstance(x, (int, float)) and not isinstance(x, bool) for x in v):
        raise ConfigError(f"bad value for '{key}' in layer")
    return np.array(v, dtype=np.float64).astype(np.float32)


def loads(text: str) -> list[CheckpointLayer]:
    """checkpoint_from_json(json::parse(text)) (serialize.hpp:137-190)."""
    try:
        j = json.loads(text, parse_constant=_no_constants)
    except json.JSONDecodeError as e:
        raise ConfigError(f"checkpoint is not valid JSON: {e}") from None
    if not isinstance(j, dict):
        raise ConfigError("checkpoint must be a JSON object")
    for k in j:
        if k != "layers":
            raise ConfigError(f"unknown key '{k}' in checkpoint")
    if not isinstance(j.get("layers"), list):
        raise ConfigError("checkpoint must contain a layers array")
    out = []
    for lj in j["layers"]:
        if not isinstance(lj, dict):
            raise ConfigError("checkpoint layer must be a JSON object")
        for k in lj:
            if k not in LAYER_KEYS:
                raise ConfigError(f"unknown key '{k}' in checkpoint layer")
        layer_id = _required(lj, "layer_id", "layer")
        if not isinstance(layer_id, str):
            raise ConfigError("bad value for 'layer_id' in layer")
        shape = _uints(_required(lj, "shape", "layer"), "shape", 64)
        dense_len = 1
        for e in shape:
            dense_len *= e
        idx = _uints(_required(lj, "indices", "layer"), "indices", 32)
        for k in range(len(idx)):
            if idx[k] >= dense_len or (k > 0 and idx[k] <= idx[k - 1]):
                raise ConfigError(f"checkpoint indices must be strictly ascending and in range: {layer_id}")
        theta = _f32s(_required(lj, "theta32", "layer"), "theta32")
        m = _f32s(_required(lj, "adam_m", "layer"), "adam_m")
        v = _f32s(_required(lj, "adam_v", "layer"), "adam_v")
        if not (theta.size == m.size == v.size == len(idx)):
            raise ConfigError(f"checkpoint buffer length mismatch: {layer_id}")
        if any(e == 0 for e in shape):  # Tensor extents must be positive (tensor.hpp:65)
            raise DimensionError("tensor extents must be positive")
        if dense_len > (1 << 32):  # u32 local indices (prune.hpp:24); the reference fails to allocate
            raise DimensionError(f"layer too large for 32-bit indices: {layer_id}")
        out.append(CheckpointLayer(layer_id, tuple(shape), np.array(idx, dtype=np.uint32), theta, m, v))
    return out


# ---------------------------------------------------------------------------
# Pruned index sets <-> JSON: [{layer_id, dense_len, indices}]
# (serialize.hpp:84-119).

def index_sets_dumps(sets) -> str:
    """index_sets_to_json(sets).dump(): `sets` are PrunedIndexSet-like objects
    (layer_id, dense_len, indices as uint32 values)."""
    out = []
    for st in sets:
        idx = np.asarray(st.indices.cpu().numpy() if hasattr(st.indices, "cpu") else st.indices)
        if idx.dtype.itemsize == 4 and idx.dtype.kind in "iu":
            idx = idx.view(np.uint32)  # int32 storage of uint32 values (torch has no uint32)
        elif idx.dtype.kind in "iu" or idx.size == 0:
            idx = idx.astype(np.int64)  # wider integer storage: values, not bit patterns
            if idx.size and (idx.min() < 0 or idx.max() >= (1 << 32)):
                raise ParameterError("index values must fit uint32")
        else:
            raise ParameterError(f"indices must be an integer array, got {idx.dtype}")
        idx = ",".join(str(int(i)) for i in idx.tolist())
        out.append(f'{{"dense_len":{int(st.dense_len)},"indices":[{idx}],'
                   f'"layer_id":{json.dumps(str(st.layer_id), ensure_ascii=False)}}}')
    return "[" + ",".join(out) + "]"


def index_sets_loads(text: str) -> list[tuple[str, int, np.ndarray]]:
    """index_sets_from_json(json::parse(text)): (layer_id, dense_len, uint32
    indices) per set, validated as the reference does (ConfigError)."""
    try:
        arr = json.loads(text, parse_constant=_no_constants)
    except json.JSONDecodeError as e:
        raise ConfigError(f"index sets are not valid JSON: {e}") from None
    if not isinstance(arr, list):
        raise ConfigError("index sets must be a JSON array")
    out = []
    for j in arr:
        if not isinstance(j, dict):
            raise ConfigError("index set must be a JSON object")
        for k in j:
            if k not in ("layer_id", "dense_len", "indices"):
                raise ConfigError(f"unknown key '{k}' in index set")
        layer_id = _required(j, "layer_id", "index set")
        if not isinstance(layer_id, str):
            raise ConfigError("bad value for 'layer_id' in index set")
        dense_len = _uint(_required(j, "dense_len", "index set"), "dense_len", 64)
        idx = _uints(_required(j, "indices", "index set"), "indices", 32)
        for k in range(len(idx)):
            if idx[k] >= dense_len or (k > 0 and idx[k] <= idx[k - 1]):
                raise ConfigError(f"indices must be strictly ascending and in range: {layer_id}")
        out.append((layer_id, dense_len, np.array(idx, dtype=np.uint32)))
    return out
