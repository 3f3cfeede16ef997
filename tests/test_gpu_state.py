"""GPU: state formats and accounting around the step path.

* binary checkpoint = the fields of the reference's JSON checkpoint
  (serialize.hpp:120-190) + the Adam scalars; load rebuilds theta16 by
  downcast+expand (serialize.hpp:184-186) and resumes bit-exactly;
* load errors map to ConfigError, as checkpoint_from_json;
* the memory report's reference accounting equals the reference library's
  measured_bytes (store.hpp:129-147) on the same state."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def T(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint16:
        a = a.view(np.int16)
    elif a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a.copy()).cuda()


@pytest.fixture(scope="module")
def S(cuda):
    from paper_2302_05045_b200 import samo
    return samo


def _model(S, g):
    dense_len = g["dense_len"].astype(np.int64)
    L = len(dense_len)
    sets = [S.PrunedIndexSet(f"l{l}", int(dense_len[l]), T(g[f"idx{l}"])) for l in range(L)]
    m = S.SamoModel.from_index_sets(sets, [(int(d),) for d in dense_len], 1024)
    for l in range(L):
        m.init_layer(l, T(g[f"val{l}"]))
    m.set_config(S.OptimizerConfig(learning_rate=1e-2, loss_scale=1024.0))
    return m, L


def _state(m, L):
    out = {}
    for l in range(L):
        for k in ("theta32", "adam_m", "adam_v", "indices"):
            out[f"{k}{l}"] = m.read(l, k).cpu().numpy().view(np.uint32)
        out[f"theta16{l}"] = m.read(l, "theta16").cpu().numpy().view(np.uint16)
    r = m.step_record()
    out["rec"] = (r.t, r.skipped_steps, r.beta1_pow, r.beta2_pow)
    return out


def test_checkpoint_round_trip_and_resume(S, golden, tmp_path):
    g = golden("step")
    m, L = _model(S, g)
    for s in range(3):  # includes the skipped step 2
        m.set_grads([T(g[f"s{s}_grad{l}"]) for l in range(L)])
        m.step()
    path = tmp_path / "state.samo"
    m.save(str(path))
    m2 = S.SamoModel.load(str(path), tile_elems=1024)
    a, b = _state(m, L), _state(m2, L)
    assert a.keys() == b.keys()
    for k in a:
        if k == "rec":
            assert a[k] == b[k]
        else:
            assert np.array_equal(a[k], b[k]), k
    m2.check_invariants()
    # resume: the next step is identical on the original and the reloaded state
    for mm in (m, m2):
        mm.set_config(S.OptimizerConfig(learning_rate=1e-2, loss_scale=1024.0))
        mm.set_grads([T(g[f"s3_grad{l}"]) for l in range(L)])
        mm.step()
    a, b = _state(m, L), _state(m2, L)
    for k in a:
        if k != "rec":
            assert np.array_equal(a[k], b[k]), k
    for l in range(L):
        assert np.array_equal(a[f"theta32{l}"], g[f"s3_theta32{l}"].view(np.uint32))


def test_checkpoint_errors(S, golden, tmp_path):
    g = golden("step")
    m, L = _model(S, g)
    path = tmp_path / "state.samo"
    m.save(str(path))
    raw = path.read_bytes()
    (tmp_path / "short.samo").write_bytes(raw[: len(raw) // 2])
    with pytest.raises(S.ConfigError):
        S.SamoModel.load(str(tmp_path / "short.samo"))
    (tmp_path / "magic.samo").write_bytes(b"NOTSAMO!" + raw[8:])
    with pytest.raises(S.ConfigError):
        S.SamoModel.load(str(tmp_path / "magic.samo"))
    # swap two indices of layer 0 -> not ascending (serialize.hpp:156-163)
    hdr = 8 + 4 * 4 + 32 + 16 * L
    arr = bytearray(raw)
    i0 = np.frombuffer(raw, dtype=np.uint32, count=2, offset=hdr).copy()
    arr[hdr:hdr + 8] = i0[::-1].tobytes()
    (tmp_path / "order.samo").write_bytes(bytes(arr))
    with pytest.raises(S.ConfigError):
        S.SamoModel.load(str(tmp_path / "order.samo"))


def test_memory_report_matches_reference_measured_bytes(S, golden):
    from oracle.oracle import REF_SO, Cfg, RefLib, RefSession
    if not REF_SO.exists():
        pytest.skip("reference library not built")
    g = golden("step")
    m, L = _model(S, g)
    rep = m.memory()
    dense_len = g["dense_len"].astype(np.int64)
    idx = [g[f"idx{l}"] for l in range(L)]
    sess = RefSession(RefLib(), dense_len, idx, [np.zeros(len(i), np.float32) for i in idx], Cfg())
    dummy_steady, dummy_peak = 2 * 1 + 22 * 1, 2 * 1 + 24 * 1  # the shim's 1x1 driver layer
    assert rep["reference_steady_bytes"] == sess.ref.lib.ref_session_measured_bytes(sess.h, 0) - dummy_steady
    assert rep["reference_peak_bytes"] == sess.ref.lib.ref_session_measured_bytes(sess.h, 1) - dummy_peak
    assert rep["device_bytes"] >= rep["theta16_bytes"] + rep["compressed_state_bytes"]
    sess.close()


def test_json_checkpoint_round_trip(S, golden):
    """JSON checkpoint in the reference's schema (serialize.hpp:121-190):
    to_checkpoint_json of a stepped model loads back (from_checkpoint_json)
    with the same indices, theta32, m, v and the rebuilt theta16, bit for bit;
    the step scalars start afresh, as a trainer built on loaded state does.
    When oracle/_ref has the JSON entry point, the reference itself accepts
    the text too."""
    from paper_2302_05045_b200 import checkpoint_json as cj
    g = golden("step")
    m, L = _model(S, g)
    for s in range(2):
        m.set_grads([T(g[f"s{s}_grad{l}"]) for l in range(L)])
        m.step()
    text = m.to_checkpoint_json()
    assert [l.layer_id for l in cj.loads(text)] == [f"l{l}" for l in range(L)]
    m2 = S.SamoModel.from_checkpoint_json(text, tile_elems=1024)
    a, b = _state(m, L), _state(m2, L)
    for k in a:
        if k != "rec":
            assert np.array_equal(a[k], b[k]), k
    assert b["rec"][0] == 0 and b["rec"][2] == 1.0 and b["rec"][3] == 1.0
    m2.check_invariants()
    from oracle.oracle import REF_SO, RefLib
    if REF_SO.exists():
        ref = RefLib()
        if ref.has_json:
            rc, back = ref.checkpoint_json_roundtrip(text)
            assert rc == 0 and len(cj.loads(back)) == L
