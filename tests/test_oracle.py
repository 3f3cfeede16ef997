"""CPU: pins the oracle (oracle/samo_oracle.c) against the reference.

Two anchors: (1) the reference's own known-answer tests, restated from
proj/tests/{half,store,prune,train}_test.cpp; (2) golden vectors produced by
the unmodified reference headers (tests/golden/make_golden.py).
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from oracle.oracle import Cfg, StepState


def bits(x):
    return np.asarray(x, dtype=np.float32).view(np.uint32)


# --------------------------------------------------------------------------
# half_test.cpp

def test_half_spec_examples(oracle):  # half_test.cpp:54-59
    assert oracle.h2f(oracle.f2h([1.0, 2049.0, 0.5])).tolist() == [1.0, 2048.0, 0.5]


def test_half_exhaustive_round_trip(oracle):  # half_test.cpp:61-68
    h = np.arange(65536, dtype=np.uint16)
    finite = (h & 0x7C00) != 0x7C00
    assert np.array_equal(oracle.f2h(oracle.h2f(h[finite])), h[finite])


def test_half_overflow_underflow_edges(oracle):  # half_test.cpp:83-94
    cases = {65504.0: 0x7BFF, 65519.996: 0x7BFF, 65520.0: 0x7C00, 1e10: 0x7C00, -1e10: 0xFC00,
             2.0**-24: 0x0001, 2.0**-25: 0x0000, -0.0: 0x8000}
    got = oracle.f2h(np.array(list(cases), dtype=np.float32))
    assert got.tolist() == list(cases.values())
    nxt = np.nextafter(np.float32(2.0**-25), np.float32(1.0))
    assert oracle.f2h([nxt]).tolist() == [0x0001]


def test_half_inf_nan(oracle):  # half_test.cpp:70-81
    assert oracle.f2h(oracle.h2f(np.array([0x7C00, 0xFC00], np.uint16))).tolist() == [0x7C00, 0xFC00]
    nan_h = oracle.f2h([np.nan])[0]
    assert (nan_h & 0x7C00) == 0x7C00 and (nan_h & 0x3FF) != 0
    assert math.isnan(oracle.h2f(np.array([0x7E01], np.uint16))[0])


def test_half_golden(oracle, golden):
    g = golden("half")
    assert np.array_equal(oracle.f2h(g["f2h_in"]), g["f2h_out"])
    assert np.array_equal(bits(oracle.h2f(g["h2f_in"])), g["h2f_out_bits"])


# --------------------------------------------------------------------------
# store_test.cpp

def test_compress_by_definition(oracle):  # store_test.cpp:29-33
    d = np.array([1, 2, 3, 4], np.float32)
    assert oracle.compress(d, np.array([0, 3])).tolist() == [1.0, 4.0]


def test_compress_identity_and_length_error(oracle):  # store_test.cpp:35-40, 60-64
    d = np.array([1, 2, 3, 4], np.float32)
    assert oracle.compress(d, np.arange(4)).tolist() == [1, 2, 3, 4]
    with pytest.raises(ValueError):
        oracle.compress(np.zeros(3, np.float32), np.array([0]), ind_dense_len=4)


def test_expand_by_definition_and_empty(oracle):  # store_test.cpp:66-77
    got = oracle.expand(np.array([1, 4], np.float32), np.array([0, 3]), (2, 2))
    assert got.tolist() == [[1, 0], [0, 4]]
    assert oracle.expand(np.array([], np.float32), np.array([], np.uint32), (4,)).tolist() == [0] * 4


def test_store_golden_round_trips(oracle, golden):  # store_test.cpp:79-108 shape
    g = golden("store")
    off_d = off_i = 0
    for t, (n, k) in enumerate(g["rt_meta"].astype(np.int64)):
        dense = g["rt_dense"][off_d:off_d + n]
        idx = g["rt_idx"][off_i:off_i + k]
        off_d += n
        off_i += k
        vals = oracle.compress(dense, idx)
        assert np.array_equal(vals, g[f"rt{t}_vals"])
        exp = oracle.expand(vals, idx, (int(n),))
        assert np.array_equal(exp, g[f"rt{t}_exp"])
        assert np.array_equal(oracle.compress(exp, idx), vals)


# --------------------------------------------------------------------------
# prune_test.cpp

def test_prune_kats(oracle):
    assert oracle.magnitude_prune([[3.0, -1.0, 0.5, -4.0]], [True], 0.5)[0].tolist() == [0, 3]
    assert oracle.magnitude_prune([[0.1, -0.2, 0.0]], [True], 0.0)[0].tolist() == [0, 1, 2]
    assert oracle.magnitude_prune([[1.0] * 4], [True], 0.5)[0].tolist() == [0, 1]
    for p in (1.0, -0.1):
        with pytest.raises(ValueError):
            oracle.magnitude_prune([[1.0]], [True], p)
    sets = oracle.magnitude_prune([[5, 1, 2, 3], [0, 0]], [True, False], 0.75)
    assert len(sets[0]) == 1 and sets[1].tolist() == [0, 1]
    big, small = [10, 9, 8, 7], [1, 0.9, 0.8, 0.7]
    g = oracle.magnitude_prune([big, small], [True, True], 0.5, scope=1)
    assert g[0].tolist() == [0, 1, 2, 3] and g[1].tolist() == []
    pl = oracle.magnitude_prune([big, small], [True, True], 0.5, scope=0)
    assert len(pl[0]) == 2 and len(pl[1]) == 2


def test_prune_count_rounding(oracle):  # prune_test.cpp:120-147
    rng = np.random.default_rng(23)
    for _ in range(200):
        num = int(rng.integers(0, 20))
        n = int(rng.integers(1, 51))
        want = (2 * (20 - num) * n + 20) // 40
        assert oracle.unpruned_count(num / 20.0, n) == want


def test_prune_golden(oracle, golden):
    g = golden("prune")
    for c, row in enumerate(g["cases"]):
        L, p = int(row[0]), float(row[1])
        prunable = [bool(x) for x in row[2:2 + L]]
        vals = [g[f"c{c}_val{l}"] for l in range(L)]
        for scope in (0, 1):
            got = oracle.magnitude_prune(vals, prunable, p, scope)
            for l in range(L):
                assert np.array_equal(got[l], g[f"c{c}_s{scope}_idx{l}"]), (c, scope, l)


def test_prune_golden_big(oracle, golden):
    g = golden("prune")
    vals = oracle.mt64_uniform(int(g["big_seed"][0]), 4096 * 1024, 1.0 / 64.0)
    got = oracle.magnitude_prune([vals], [True], 0.9)[0]
    assert np.array_equal(got, g["big_idx"])


# --------------------------------------------------------------------------
# train_test.cpp / adam

def test_adam_scalar_oracle(oracle):  # train_test.cpp:156-180
    th, m, v = (np.array([x], np.float32) for x in (0.5, 0.0, 0.0))
    g = np.array([1.0], np.float32)
    b1 = np.float32(1.0) - np.float32(0.9)
    b2 = np.float32(1.0) - np.float32(0.999)
    oracle.adam_update(th, m, v, g, Cfg(lr=0.1, loss_scale=1.0), float(b1), float(b2))
    assert abs(th[0] - 0.4) <= 1e-6


def test_adam_golden(oracle, golden):
    g = golden("adam")
    for tag in ("plain", "wd", "late"):
        c = g[f"{tag}_cfg"]
        cfg = Cfg(lr=float(c[0]), beta1=float(c[1]), beta2=float(c[2]), eps=float(c[3]),
                  loss_scale=float(c[4]), wd=float(c[5]))
        th, m, v = g["th"].copy(), g["m"].copy(), g["v"].copy()
        oracle.adam_update(th, m, v, g["g"], cfg, float(c[6]), float(c[7]))
        assert np.array_equal(bits(th), bits(g[f"{tag}_th"]))
        assert np.array_equal(bits(m), bits(g[f"{tag}_m"]))
        assert np.array_equal(bits(v), bits(g[f"{tag}_v"]))


def test_optimizer_step_golden(oracle, golden):
    """Five reference optimizer steps (one skipped on +inf), bit-exact."""
    g = golden("step")
    dense_len = g["dense_len"].astype(np.int64)
    L = len(dense_len)
    idx = [g[f"idx{l}"] for l in range(L)]
    nnz = np.array([len(i) for i in idx], np.uint64)
    arena = np.concatenate(idx).astype(np.uint32)
    theta = np.concatenate([oracle.compress(g[f"val{l}"], idx[l]) for l in range(L)])
    m, v, g32 = (np.zeros_like(theta) for _ in range(3))
    t16 = [np.zeros(int(d), np.uint16) for d in dense_len]
    st = StepState()
    cfg = Cfg(lr=1e-2, loss_scale=1024.0)
    for s in range(int(g["steps"][0])):
        applied = oracle.optimizer_step(dense_len, nnz, arena, [g[f"s{s}_grad{l}"] for l in range(L)],
                                        theta, m, v, g32, t16, cfg, st)
        assert applied == bool(g[f"s{s}_applied"][0])
        assert st.skipped == int(g[f"s{s}_skipped"][0])
        assert np.float32(st.grad_norm) == g[f"s{s}_norm"][0]
        k0 = 0
        for l in range(L):
            n = int(nnz[l])
            assert np.array_equal(bits(theta[k0:k0 + n]), bits(g[f"s{s}_theta32{l}"]))
            assert np.array_equal(bits(m[k0:k0 + n]), bits(g[f"s{s}_adam_m{l}"]))
            assert np.array_equal(bits(v[k0:k0 + n]), bits(g[f"s{s}_adam_v{l}"]))
            assert np.array_equal(t16[l], g[f"s{s}_theta16{l}"])
            k0 += n


def test_mt64_matches_std_engine(oracle):
    # first outputs of std::mt19937_64 default seed 5489 (C++ standard [rand.predef])
    st = oracle.mt64_raw(5489, 10000)
    assert int(st[-1]) == 9981545732273789042


def test_dp_sum_order(oracle):
    a = np.array([1e8, 1.0, -1.0], np.float32)
    b = np.array([1.0, 1e8, 1.0], np.float32)
    s, absum = oracle.dp_sum([a, b])
    assert s.tolist() == [np.float32(1e8) + np.float32(1.0), np.float32(1.0) + np.float32(1e8), 0.0]
    assert absum.tolist() == [1e8 + 1, 1e8 + 1, 2.0]


@pytest.mark.parametrize("batch,n_in,n_out", [(1, 8, 8), (64, 24, 40), (576, 16, 32), (7, 3, 5)])
def test_dw_matmul_matches_reference(oracle, batch, n_in, n_out):
    """The oracle's restatement of matmul(transpose(x), dy) (train.hpp:304,
    tensor.hpp:88-105) equals the reference library bit for bit."""
    from oracle.oracle import REF_SO, RefLib
    if not REF_SO.exists():
        pytest.skip("reference library not built")
    rng = np.random.default_rng(batch + n_in)
    x = oracle.f2h(rng.uniform(-1, 1, batch * n_in).astype(np.float32)).reshape(batch, n_in)
    dy = oracle.f2h((rng.uniform(-1, 1, batch * n_out) * 1024 / batch).astype(np.float32)).reshape(batch, n_out)
    rc, want = RefLib().dw_matmul(x, dy)
    assert rc == 0
    assert np.array_equal(oracle.dw_matmul(x, dy), want)


def test_bf16_widening_exhaustive(oracle):
    """or_bf16_to_float: every bf16 pattern is the top half of its binary32
    (exact widening, NaN payloads kept)."""
    h = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    got = oracle.bf16_to_float(h)
    assert np.array_equal(got.view(np.uint32), h.astype(np.uint32) << 16)


def test_bf16_step_equals_f16_step_on_common_values(oracle):
    """Gradients representable in both 16-bit types (binary16 patterns with
    the low 3 mantissa bits clear, normal range) give bit-identical steps
    through the binary16 and the bfloat16 decode."""
    from oracle.oracle import Cfg, StepState
    rng = np.random.default_rng(4)
    d = 5000
    idx = np.sort(rng.choice(d, 900, replace=False)).astype(np.uint32)
    v0 = (rng.standard_normal(d) * 0.05).astype(np.float32)
    h16 = oracle.f2h((rng.standard_normal(d) * 8.0).astype(np.float32)) & np.uint16(0xFFF8)
    h16[(h16 & 0x7C00) == 0] = 0  # no binary16 subnormals
    f = oracle.h2f(h16)
    hb = (f.view(np.uint32) >> 16).astype(np.uint16)
    assert np.array_equal((hb.astype(np.uint32) << 16).view(np.float32), f)
    out = []
    for grads, bf in ((h16, False), (hb, True)):
        theta = oracle.compress(v0, idx)
        m, v, g32 = (np.zeros_like(theta) for _ in range(3))
        t16 = [np.zeros(d, np.uint16)]
        st = StepState()
        for _ in range(2):
            oracle.optimizer_step([d], [len(idx)], idx, [grads], theta, m, v, g32, t16, Cfg(), st, grad_bf16=bf)
        out.append((theta.view(np.uint32).copy(), v.view(np.uint32).copy(), t16[0].copy()))
    for a, b in zip(*out):
        assert np.array_equal(a, b)
