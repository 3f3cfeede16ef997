"""CPU check of the NCCL-exchange parity checker (test_gpu_dp.py's
_check_nccl_tolerance): replicas built by the oracle with other fp32
summation orders than rank-ascending (descending, pairwise tree — the
shapes of NCCL's ring and tree/NVLS reductions) must pass, and a gradient or
a weight moved outside the stated bounds must fail."""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))


def _sum(parts, order):
    if order == "tree":
        while len(parts) > 1:
            nxt = [(parts[i] + parts[i + 1]).astype(np.float32) for i in range(0, len(parts) - 1, 2)]
            if len(parts) % 2:
                nxt.append(parts[-1])
            parts = nxt
        return parts[0]
    acc = np.zeros_like(parts[0])
    for p in (reversed(parts) if order == "desc" else parts):
        acc = (acc + p).astype(np.float32)
    return acc


def _replicas(oracle, world, order, steps=4):
    """What an allreduce exchange that sums in `order` would leave on every
    rank, in dp_worker.py's output format."""
    os.environ["SAMO_DP_STEPS"] = str(steps)
    import importlib
    import dp_worker as W
    W = importlib.reload(W)
    from oracle.oracle import Cfg
    vals, sets, grads = W.inputs(oracle, world)
    L = len(W.DENSE_LEN)
    cfg = Cfg(lr=1e-2)
    inv = np.float32(1.0) / np.float32(1024.0) * (np.float32(1.0) / np.float32(world))
    theta = [oracle.compress(v, s) for v, s in zip(vals, sets)]
    m = [np.zeros_like(t) for t in theta]
    v = [np.zeros_like(t) for t in theta]
    b1p = b2p = np.float32(1.0)
    t = skipped = 0
    rr = {}
    for s in range(steps):
        g = []
        for l in range(L):
            parts = [(oracle.h2f(oracle.compress(grads[(q, s, l)], sets[l])) * inv).astype(np.float32)
                     for q in range(world)]
            g.append(_sum(parts, order))
            rr[f"g32_{s}_{l}"] = g[-1]
        if not all(np.all(np.isfinite(x)) for x in g):
            skipped += 1
            continue
        t += 1
        b1p = np.float32(b1p * np.float32(0.9))
        b2p = np.float32(b2p * np.float32(0.999))
        for l in range(L):
            oracle.adam_update(theta[l], m[l], v[l], g[l], cfg, float(np.float32(1) - b1p),
                               float(np.float32(1) - b2p))
    n = sum(len(x) for x in theta)
    rr.update({"t": np.array([t]), "skipped": np.array([skipped]),
               "shard": np.array([[0, n]], np.uint64),
               "k_off": np.cumsum([0] + [len(x) for x in theta])[:-1].astype(np.uint64)})
    for l in range(L):
        rr[f"theta32{l}"], rr[f"adam_m{l}"], rr[f"adam_v{l}"] = theta[l], m[l], v[l]
        rr[f"theta16_{l}"] = oracle.expand(oracle.f2h(theta[l]), sets[l], (W.DENSE_LEN[l],))
    return [rr] * world


@pytest.mark.parametrize("G,order", [(3, "desc"), (4, "desc"), (4, "tree"), (8, "tree"), (8, "desc")])
def test_other_summation_orders_pass(oracle, G, order):
    from test_gpu_dp import _check_nccl_tolerance
    _check_nccl_tolerance(_replicas(oracle, G, order), oracle, G, "overlap")


def test_out_of_bound_results_fail(oracle):
    from test_gpu_dp import _check_nccl_tolerance
    r = _replicas(oracle, 4, "desc")
    bad = dict(r[0])
    x = bad["g32_1_0"].copy()
    x[7] *= np.float32(1.0001)  # far outside (G-1) 2^-24 sum|g_r|
    bad["g32_1_0"] = x
    with pytest.raises(AssertionError):
        _check_nccl_tolerance([bad] * 4, oracle, 4, "overlap")
    with pytest.raises(AssertionError, match="replicas differ"):
        _check_nccl_tolerance([bad] + r[1:], oracle, 4, "overlap")
    bad = dict(r[0])
    y = bad["theta320"].copy()
    y[3] = np.nextafter(y[3], np.float32(np.inf))  # one ulp off the replayed update
    bad["theta320"] = y
    with pytest.raises(AssertionError):
        _check_nccl_tolerance([bad] * 4, oracle, 4, "overlap")
