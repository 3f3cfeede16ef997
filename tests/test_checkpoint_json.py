"""CPU: JSON checkpoints in the reference's schema (serialize.hpp:121-190)
against the reference's own checkpoint_from_json / checkpoint_to_json
(oracle/_ref, built with nlohmann/json when available):

* our dump loads in the reference, and the reference's re-dump loads in ours
  with every value bit-identical; the texts agree except for Grisu2's
  occasional alternative last digit, so values are compared, not bytes;
* every malformed checkpoint the reference rejects, we reject with the
  same error class (ConfigError / DimensionError), and vice versa.
"""
from __future__ import annotations

import json

import numpy as np
import pytest

from oracle.oracle import REF_SO, RefLib
from paper_2302_05045_b200 import checkpoint_json as cj
from paper_2302_05045_b200._abi import ConfigError, DimensionError, SamoError


@pytest.fixture(scope="module")
def ref():
    if not REF_SO.exists():
        pytest.skip("oracle/_ref not built")
    r = RefLib()
    if not r.has_json:
        pytest.skip("oracle/_ref built without nlohmann/json")
    return r


def _layers(seed):
    rng = np.random.default_rng(seed)
    out = []
    for l, shape in enumerate([(7, 5), (64,), (3, 4, 5)]):
        n = int(np.prod(shape))
        idx = np.flatnonzero(rng.random(n) < 0.4).astype(np.uint32)
        k = idx.size
        vals = [(rng.standard_normal(k) * 10.0 ** rng.integers(-30, 30, k)).astype(np.float32) for _ in range(3)]
        vals[0][:3] = np.array([0.1, -0.0, 1e-45], dtype=np.float32)[: min(3, k)]
        out.append(cj.CheckpointLayer(f"layer{l}", shape, idx, *vals))
    return out


@pytest.mark.parametrize("seed", range(5))
def test_round_trip_through_the_reference(ref, seed):
    layers = _layers(seed)
    ours = cj.dumps(layers)
    rc, theirs = ref.checkpoint_json_roundtrip(ours)
    assert rc == 0
    assert len(theirs) == pytest.approx(len(ours), rel=0.01)  # same layout, up to Grisu2 digits
    back = cj.loads(theirs)
    for a, b in zip(layers, back):
        assert a.layer_id == b.layer_id and tuple(a.shape) == b.shape
        assert np.array_equal(a.indices, b.indices)
        for k in ("theta32", "adam_m", "adam_v"):
            assert np.array_equal(getattr(a, k).view(np.uint32), getattr(b, k).view(np.uint32))


def _mutations():
    base = json.loads(cj.dumps(_layers(0)))
    cases = {}

    def case(name, fn):
        j = json.loads(json.dumps(base))
        fn(j)
        cases[name] = json.dumps(j)

    case("unknown_top_key", lambda j: j.update(extra=1))
    case("unknown_layer_key", lambda j: j["layers"][0].update(grad16=[]))
    case("missing_theta", lambda j: j["layers"][1].pop("theta32"))
    case("descending_indices", lambda j: j["layers"][0].update(indices=j["layers"][0]["indices"][::-1]))
    case("index_out_of_range", lambda j: j["layers"][1]["indices"].__setitem__(-1, 64))
    case("length_mismatch", lambda j: j["layers"][2]["adam_m"].pop())
    case("null_value", lambda j: j["layers"][0]["adam_v"].__setitem__(0, None))
    case("string_value", lambda j: j["layers"][0]["theta32"].__setitem__(0, "x"))
    case("layer_id_not_string", lambda j: j["layers"][0].update(layer_id=3))
    case("layers_not_array", lambda j: j.update(layers={}))
    case("not_object", lambda j: None)
    cases["not_object"] = "[1, 2]"
    case("zero_extent", lambda j: j["layers"][1].update(shape=[0], indices=[], theta32=[], adam_m=[], adam_v=[]))
    case("empty_ok", lambda j: j.update(layers=[]))
    # nlohmann's get<uintN_t>() casts: integral floats and truncated fractions
    # are accepted, negative integers wrap (and then fail the range check)
    case("float_shape", lambda j: j["layers"][0].update(shape=[7.0, 5.0]))
    case("fractional_shape", lambda j: j["layers"][0].update(shape=[7.9, 5.2]))
    case("float_index", lambda j: j["layers"][1]["indices"].__setitem__(0, float(j["layers"][1]["indices"][0])))
    case("fractional_index", lambda j: j["layers"][1]["indices"].__setitem__(0, j["layers"][1]["indices"][0] + 0.5))
    case("negative_index", lambda j: j["layers"][1]["indices"].__setitem__(0, -1))
    case("negative_shape", lambda j: j["layers"][1].update(shape=[-64]))
    case("bool_index", lambda j: j["layers"][1]["indices"].__setitem__(0, True))
    return cases


@pytest.mark.parametrize("name,text", sorted(_mutations().items()))
def test_same_rejections_as_the_reference(ref, name, text):
    rc, theirs = ref.checkpoint_json_roundtrip(text)
    if rc == 0:  # accepted by both, read to the same values
        got, want = cj.loads(text), cj.loads(theirs)
        assert [(a.layer_id, tuple(a.shape), a.indices.tolist()) for a in got] == \
            [(b.layer_id, tuple(b.shape), b.indices.tolist()) for b in want]
        return
    # 99: the reference fails outside its own error classes (a wrapped
    # negative extent makes a 2^64-element tensor); any SamoError will do
    want = {5: ConfigError, 1: DimensionError, 99: SamoError}[rc]
    with pytest.raises(want):
        cj.loads(text)


def test_index_sets_round_trip_through_the_reference(ref, oracle):
    """index_sets_to_json / index_sets_from_json (serialize.hpp:84-119): K0's
    output format for masks, byte for byte (integers only) both ways."""
    from types import SimpleNamespace
    rng = np.random.default_rng(3)
    vals = [rng.standard_normal(n).astype(np.float32) for n in (300, 1, 5000)]
    sets = [SimpleNamespace(layer_id=f"w{l}", dense_len=v.size, indices=s)
            for l, (v, s) in enumerate(zip(vals, oracle.magnitude_prune(vals, [True, False, True], 0.9)))]
    ours = cj.index_sets_dumps(sets)
    rc, theirs = ref.index_sets_json_roundtrip(ours)
    assert rc == 0 and theirs == ours
    back = cj.index_sets_loads(theirs)
    assert [(b[0], b[1]) for b in back] == [(s.layer_id, s.dense_len) for s in sets]
    for b, s in zip(back, sets):
        assert np.array_equal(b[2], s.indices)


@pytest.mark.parametrize("text", [
    '{"layer_id":"a"}', '[{"layer_id":"a","dense_len":4,"indices":[0,2],"x":1}]',
    '[{"layer_id":"a","dense_len":4,"indices":[2,0]}]', '[{"layer_id":"a","dense_len":4,"indices":[4]}]',
    '[{"layer_id":"a","indices":[0]}]', '[{"layer_id":1,"dense_len":4,"indices":[0]}]',
    '[{"layer_id":"a","dense_len":4,"indices":[0,1]}]', '[]',
    '[{"layer_id":"a","dense_len":4.7,"indices":[0,1]}]', '[{"layer_id":"a","dense_len":4,"indices":[1.0,2.5]}]',
    '[{"layer_id":"a","dense_len":4,"indices":[-1]}]', '[{"layer_id":"a","dense_len":-1,"indices":[0,7]}]',
    '[{"layer_id":"a","dense_len":4,"indices":[true]}]', '[{"layer_id":"a","dense_len":"4","indices":[0]}]'])
def test_index_sets_same_rejections_as_the_reference(ref, text):
    rc, theirs = ref.index_sets_json_roundtrip(text)
    if rc == 0:  # accepted by both, read to the same values
        from types import SimpleNamespace
        got = cj.index_sets_loads(text)
        assert cj.index_sets_dumps([SimpleNamespace(layer_id=a, dense_len=d, indices=i) for a, d, i in got]) == theirs
        return
    with pytest.raises({5: ConfigError, 1: DimensionError}[rc]):
        cj.index_sets_loads(text)


def test_index_sets_dump_takes_values_of_any_integer_dtype():
    """int64 / Python-int indices are values: never split into
    32-bit words; out-of-range and non-integer arrays are refused."""
    from types import SimpleNamespace
    from paper_2302_05045_b200._abi import ParameterError
    want = '[{"dense_len":10,"indices":[1,4,9],"layer_id":"a"}]'
    for idx in ([1, 4, 9], np.array([1, 4, 9], np.int64), np.array([1, 4, 9], np.uint32),
                np.array([1, 4, 9], np.int32), np.array([1, 4, 9], np.uint16)):
        assert cj.index_sets_dumps([SimpleNamespace(layer_id="a", dense_len=10, indices=idx)]) == want
    big = np.array([0, 1 << 32], np.int64)
    with pytest.raises(ParameterError):
        cj.index_sets_dumps([SimpleNamespace(layer_id="a", dense_len=1 << 33, indices=big)])
    with pytest.raises(ParameterError):
        cj.index_sets_dumps([SimpleNamespace(layer_id="a", dense_len=10, indices=np.array([1.0]))])


def test_index_sets_python_api_on_cpu_tensors():
    """samo.index_sets_from_json / index_sets_to_json round trip (host tensors)."""
    from paper_2302_05045_b200 import samo
    text = '[{"dense_len":10,"indices":[1,4,9],"layer_id":"a"},{"dense_len":3,"indices":[],"layer_id":"b"}]'
    sets = samo.index_sets_from_json(text, device="cpu")
    assert [s.layer_id for s in sets] == ["a", "b"] and sets[0].indices.tolist() == [1, 4, 9]
    assert samo.index_sets_to_json(sets) == text
