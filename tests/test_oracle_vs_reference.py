"""CPU: the oracle (oracle/samo_oracle.c) against the reference itself on
random inputs — the unmodified reference headers compiled into
oracle/_ref/libsamo_ref.so (oracle/ref_shim.cpp) — beyond the fixed golden
vectors of test_oracle.py.  Every comparison is bit for bit:

* Half conversions on random fp32 bit patterns (all classes: subnormal,
  overflow, NaN payloads) — half.hpp:13-71;
* compress / expand, including length errors — store.hpp:58-87;
* adam_update over random states, edge values and weight decay —
  train.hpp:332-347;
* magnitude_prune, per-layer and global, with ties and non-prunable layers —
  prune.hpp:99-170;
* whole optimizer steps (SamoTrainer::optimizer_step, train.hpp:617-656)
  including a skipped step, over several layers.

Skipped when oracle/_ref was not built (no /root/reference on this host).
"""
from __future__ import annotations

import numpy as np
import pytest

pytest.importorskip("hypothesis")
from hypothesis import assume, given, settings, strategies as st  # noqa: E402

from oracle.oracle import REF_SO, Cfg, RefLib, RefSession, StepState  # noqa: E402

pytestmark = pytest.mark.skipif(not REF_SO.exists(), reason="oracle/_ref not built")

SETTINGS = settings(max_examples=40, deadline=None, derandomize=True)


@pytest.fixture(scope="module")
def ref():
    return RefLib()


def _bits32(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


@SETTINGS
@given(seed=st.integers(0, 2**32 - 1))
def test_half_conversions_random_bits(oracle, ref, seed):
    rng = np.random.default_rng(seed)
    w = rng.integers(0, 2**32, 4096, dtype=np.uint64).astype(np.uint32)
    w[:8] = [0x00000001, 0x33000000, 0x387FE000, 0x477FF000, 0x477FE000, 0x7F800001, 0xFFC12345, 0x80000000]
    f = w.view(np.float32)
    assert np.array_equal(oracle.f2h(f), ref.f2h(f))
    h = rng.integers(0, 65536, 4096, dtype=np.uint32).astype(np.uint16)
    assert np.array_equal(_bits32(oracle.h2f(h)), _bits32(ref.h2f(h)))


@SETTINGS
@given(dense_len=st.integers(1, 3000), density=st.floats(0.0, 1.0), seed=st.integers(0, 2**31),
       bad_len=st.booleans())
def test_compress_expand_random(oracle, ref, dense_len, density, seed, bad_len):
    rng = np.random.default_rng(seed)
    idx = np.flatnonzero(rng.random(dense_len) < density).astype(np.uint32)
    dense = rng.integers(0, 65536, dense_len, dtype=np.uint32).astype(np.uint16)
    ind_len = dense_len + 1 if bad_len else dense_len
    rc, want = ref.compress(dense, idx, ind_len)
    if rc:
        with pytest.raises(ValueError):
            oracle.compress(dense, idx, ind_len)
        return
    got = oracle.compress(dense, idx, ind_len)
    assert np.array_equal(got, want)
    rc, want_e = ref.expand(got, idx, dense_len)
    assert rc == 0
    assert np.array_equal(oracle.expand(got, idx, (dense_len,)), want_e)


_special = st.sampled_from([0.0, -0.0, 1e-45, -1e-45, 1e-38, 3.4e38, -3.4e38, 1.0, -1.0, 65504.0, 1e-8])


@SETTINGS
@given(n=st.integers(1, 257), seed=st.integers(0, 2**31), wd=st.sampled_from([0.0, 0.01, 0.1]),
       lr=st.sampled_from([1e-3, 1e-2, 0.5]), t=st.integers(1, 200), special=_special)
def test_adam_update_random(oracle, ref, n, seed, wd, lr, t, special):
    rng = np.random.default_rng(seed)
    cfg = Cfg(lr=lr, wd=wd)
    theta = (rng.standard_normal(n) * 0.1).astype(np.float32)
    m = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    v = np.abs(rng.standard_normal(n) * 1e-6).astype(np.float32)
    g = (rng.standard_normal(n) * 10.0 ** rng.integers(-8, 3, n)).astype(np.float32)
    g[0] = special
    theta[-1] = special
    b1p, b2p = np.float32(1.0), np.float32(1.0)
    for _ in range(t):  # AdamScalars::advance: repeated float multiplies
        b1p, b2p = np.float32(b1p * np.float32(0.9)), np.float32(b2p * np.float32(0.999))
    bias1, bias2 = float(np.float32(1) - b1p), float(np.float32(1) - b2p)
    a = [x.copy() for x in (theta, m, v)]
    b = [x.copy() for x in (theta, m, v)]
    oracle.adam_update(a[0], a[1], a[2], g, cfg, bias1, bias2)
    ref.adam_update(b[0], b[1], b[2], g, cfg, bias1, bias2)
    for x, y in zip(a, b):
        assert np.array_equal(_bits32(x), _bits32(y))


@SETTINGS
@given(sizes=st.lists(st.integers(0, 600), min_size=1, max_size=4).filter(lambda z: any(z) or len(z) > 1),
       seed=st.integers(0, 2**31),
       p=st.sampled_from([0.0, 0.1, 0.5, 0.9, 0.95, 0.999, 1.0]), scope=st.sampled_from([0, 1]),
       levels=st.sampled_from([0, 4, 64]), prunable_mask=st.integers(0, 15))
def test_magnitude_prune_random(oracle, ref, sizes, seed, p, scope, levels, prunable_mask):
    rng = np.random.default_rng(seed)
    vals = []
    for n in sizes:
        if levels:  # few distinct magnitudes: many ties, broken by (layer, index)
            v = rng.integers(-levels, levels + 1, n).astype(np.float32) / levels
        else:
            v = rng.standard_normal(n).astype(np.float32)
        vals.append(v)
    prunable = [bool((prunable_mask >> i) & 1) for i in range(len(sizes))]
    rc, want = ref.magnitude_prune(vals, prunable, p, scope)
    # rc 1: the reference's Tensor cannot hold a zero-length layer ("tensor
    # extents must be positive", tensor.hpp:65): not expressible there, so
    # nothing to compare (the oracle returns an empty set for one).
    assume(rc != 1)
    if rc:  # ParameterError (sparsity outside [0, 1)): the oracle raises too
        with pytest.raises(ValueError):
            oracle.magnitude_prune(vals, prunable, p, scope)
        return
    got = oracle.magnitude_prune(vals, prunable, p, scope)
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


@settings(max_examples=15, deadline=None, derandomize=True)
@given(sizes=st.lists(st.integers(1, 400), min_size=1, max_size=3), seed=st.integers(0, 2**31),
       p=st.sampled_from([0.5, 0.9]), steps=st.integers(1, 4), inf_step=st.integers(-1, 3))
def test_optimizer_steps_random(oracle, ref, sizes, seed, p, steps, inf_step):
    rng = np.random.default_rng(seed)
    vals = [(rng.standard_normal(n) * 0.05).astype(np.float32) for n in sizes]
    sets = oracle.magnitude_prune(vals, [True] * len(sizes), p)
    cfg = Cfg(lr=1e-2, wd=0.01)
    theta = [oracle.compress(v, s) for v, s in zip(vals, sets)]
    sess = RefSession(ref, sizes, sets, theta, cfg)
    try:
        th = np.concatenate(theta).astype(np.float32)
        m, v, g32 = (np.zeros_like(th) for _ in range(3))
        # make_layer_state (store.hpp:150-168): theta16 = expand(half(theta32))
        t16 = [oracle.expand(oracle.f2h(t), s_, (n,)).copy() for t, s_, n in zip(theta, sets, sizes)]
        idx = np.concatenate(sets).astype(np.uint32) if th.size else np.zeros(1, np.uint32)
        ost = StepState()
        for s in range(steps):
            grads = [oracle.f2h((rng.standard_normal(n) * 2.0**-7 * 1024.0).astype(np.float32)) for n in sizes]
            if s == inf_step and sets[0].size:
                grads[0][int(sets[0][0])] = 0x7C00  # +inf: the step is skipped (train.hpp:632-639)
            a = oracle.optimizer_step(sizes, [x.size for x in sets], idx, grads, th, m, v, g32, t16, cfg, ost)
            b = sess.step(grads)
            assert a == b
        skipped, norm = sess.counters()
        assert ost.skipped == skipped
        off = 0
        for l, n in enumerate(sizes):
            r = sess.read(l)
            k = sets[l].size
            for name, mine in (("theta32", th), ("adam_m", m), ("adam_v", v)):
                assert np.array_equal(_bits32(mine[off:off + k]), _bits32(r[name])), (name, l)
            assert np.array_equal(t16[l], r["theta16"]), l
            off += k
    finally:
        sess.close()
