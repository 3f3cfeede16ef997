"""Generates the golden vectors in tests/golden/*.npz from the REFERENCE ITSELF.

Every output below is computed by the unmodified reference headers
(/root/reference/proj/include/samo) compiled into oracle/_ref/libsamo_ref.so
by oracle/Makefile; this script only chooses inputs and records outputs.  The
fixtures pin both oracle/samo_oracle.c (tests/test_oracle.py, CPU) and the
CUDA path (tests/test_gpu_*.py) — /root/reference is not needed at test time.

    make -C oracle && python tests/golden/make_golden.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.oracle import Cfg, RefLib, RefSession  # noqa: E402

OUT = Path(__file__).resolve().parent


def half_vectors(ref: RefLib) -> dict:
    rng = np.random.default_rng(2024)
    # edge cases of half_test.cpp:54-121 plus random bit patterns
    edges = np.array([0.0, -0.0, 1.0, 2049.0, 2047.0, 2050.0, 0.1, 3.14159, 65503.5, 65504.0,
                      65519.0, 65519.996, 65520.0, 65536.0, 2.0**-14, 2.0**-15, 2.0**-24,
                      2.0**-25, 1.5 * 2.0**-24, float.fromhex("0x1.ffcp-15"), 1e-30, -1e-30, 1e30, 1e10, -1e10,
                      np.inf, -np.inf], dtype=np.float32)
    near = np.concatenate([edges, np.nextafter(edges, np.float32(1e38)),
                           np.nextafter(edges, np.float32(-1e38)), -edges])
    nans = np.array([0x7FC00000, 0x7F800001, 0xFFC00001, 0x7FBFFFFF, 0x7F802000, 0xFFFFFFFF],
                    dtype=np.uint32).view(np.float32)
    rand = rng.integers(0, 2**32, size=200_000, dtype=np.uint64).astype(np.uint32).view(np.float32)
    f = np.concatenate([near.astype(np.float32), nans, rand])
    h_all = np.arange(65536, dtype=np.uint16)
    return {"f2h_in": f, "f2h_out": ref.f2h(f), "h2f_in": h_all,
            "h2f_out_bits": ref.h2f(h_all).view(np.uint32)}


def store_vectors(ref: RefLib) -> dict:
    """compress/expand round trips in the shape of store_test.cpp:79-108."""
    rng = np.random.default_rng(43)
    out = {}
    dense_all, idx_all, meta = [], [], []
    for trial in range(300):
        nd = int(rng.integers(1, 4))
        shape = [int(rng.integers(1, 40)) for _ in range(nd)]
        n = int(np.prod(shape))
        keep = rng.integers(0, 3, size=n) != 0
        idx = np.nonzero(keep)[0].astype(np.uint32)
        x = ((rng.integers(0, 2**24, size=n).astype(np.float32) * 2.0**-24 - 0.5) * 8.0)
        xh = ref.f2h(x.astype(np.float32))
        rc, vals = ref.compress(xh, idx)
        assert rc == 0
        rc, exp = ref.expand(vals, idx, n)
        assert rc == 0
        dense_all.append(xh)
        idx_all.append(idx)
        meta.append((n, idx.size))
        out[f"rt{trial}_vals"] = vals
        out[f"rt{trial}_exp"] = exp
    out["rt_dense"] = np.concatenate(dense_all)
    out["rt_idx"] = np.concatenate(idx_all)
    out["rt_meta"] = np.array(meta, dtype=np.uint64)
    return out


def prune_vectors(ref: RefLib) -> dict:
    rng = np.random.default_rng(7)
    out = {}
    cases = []
    for c in range(60):
        L = int(rng.integers(1, 5))
        if c % 3 == 0:  # heavy ties
            vals = [(rng.integers(-6, 7, size=int(rng.integers(1, 400))) * 0.5).astype(np.float32)
                    for _ in range(L)]
        else:
            vals = [rng.standard_normal(int(rng.integers(1, 5000))).astype(np.float32)
                    for _ in range(L)]
        prunable = [bool(rng.integers(0, 4)) for _ in range(L)]
        p = float(rng.integers(0, 20)) / 20.0
        for scope in (0, 1):
            rc, sets = ref.magnitude_prune(vals, prunable, p, scope)
            assert rc == 0
            key = f"c{c}_s{scope}"
            for l, s in enumerate(sets):
                out[f"{key}_idx{l}"] = s
        for l, v in enumerate(vals):
            out[f"c{c}_val{l}"] = v
        cases.append((L, p, *[int(x) for x in prunable], *([0] * (4 - L))))
    out["cases"] = np.array(cases, dtype=np.float64)
    # one larger layer (4096x1024, p=0.9) with the init_params distribution
    big = ref.uniform_symmetric(7, 1.0 / 64.0, 4096 * 1024)
    rc, sets = ref.magnitude_prune([big], [True], 0.9, 0)
    assert rc == 0
    out["big_seed"] = np.array([7], dtype=np.uint64)
    out["big_idx"] = sets[0]
    return out


def adam_vectors(ref: RefLib) -> dict:
    rng = np.random.default_rng(5)
    n = 50_000
    th = rng.standard_normal(n).astype(np.float32)
    m = (rng.standard_normal(n) * 1e-2).astype(np.float32)
    v = (np.abs(rng.standard_normal(n)) * 1e-4).astype(np.float32)
    g = rng.standard_normal(n).astype(np.float32)
    g[:16] = [0.0, -0.0, 1e-38, -1e-38, 1e-45, 3.4e38, -3.4e38, 1.0, -1.0, 65504.0, 2.0**-24,
              1e-20, -1e-20, 1e20, 7.0, -7.0]
    out = {"th": th.copy(), "m": m.copy(), "v": v.copy(), "g": g}
    for tag, cfg, b1, b2 in (("plain", Cfg(lr=1e-3), 0.1, 0.001),
                             ("wd", Cfg(lr=3e-3, wd=0.01), 0.19, 0.001999),
                             ("late", Cfg(lr=1e-4, beta1=0.8, beta2=0.99), 0.99, 0.5)):
        t1, m1, v1 = th.copy(), m.copy(), v.copy()
        ref.adam_update(t1, m1, v1, g, cfg, b1, b2)
        out[f"{tag}_th"], out[f"{tag}_m"], out[f"{tag}_v"] = t1, m1, v1
        out[f"{tag}_cfg"] = np.array([cfg.lr, cfg.beta1, cfg.beta2, cfg.eps, cfg.loss_scale,
                                      cfg.wd, b1, b2], dtype=np.float32)
    return out


def step_vectors(ref: RefLib) -> dict:
    """Several SamoTrainer::optimizer_step calls of the unmodified reference
    (driver-layer trick), including a skipped step, on a 5-layer set."""
    from oracle.oracle import Oracle
    o = Oracle()  # only used to generate synthetic inputs (counter hash)
    rng = np.random.default_rng(11)
    dense_len = [3000, 1, 17, 8192 + 5, 40000]
    prunable = [True, False, True, True, True]
    vals = [rng.standard_normal(d).astype(np.float32) * 0.05 for d in dense_len]
    rc, sets = ref.magnitude_prune(vals, prunable, 0.9, 0)
    assert rc == 0
    th = [ref.compress(v, s)[1] for v, s in zip(vals, sets)]
    cfg = Cfg(lr=1e-2, loss_scale=1024.0, wd=0.0)
    sess = RefSession(ref, dense_len, sets, th, cfg)
    out = {"dense_len": np.array(dense_len, np.uint64), "prunable": np.array(prunable, np.uint8)}
    for l in range(len(dense_len)):
        out[f"val{l}"] = vals[l]
        out[f"idx{l}"] = sets[l]
    steps = 5
    for s in range(steps):
        grads = [o.synth_f16(0, d, 99, 1000 * s + l, 2.0**-7, 1024.0)
                 for l, d in enumerate(dense_len)]
        if s == 2:
            grads[3][100] = 0x7C00  # +inf -> the step is skipped (train.hpp:632-639)
        applied = sess.step(grads)
        out[f"s{s}_applied"] = np.array([applied], np.uint8)
        for l in range(len(dense_len)):
            out[f"s{s}_grad{l}"] = grads[l]
        sk, gn = sess.counters()
        out[f"s{s}_skipped"] = np.array([sk], np.uint64)
        out[f"s{s}_norm"] = np.array([gn], np.float32)
        for l in range(len(dense_len)):
            rd = sess.read(l)
            for k in ("theta32", "adam_m", "adam_v", "theta16"):
                out[f"s{s}_{k}{l}"] = rd[k]
    out["steps"] = np.array([steps], np.uint64)
    assert sess.check_invariants() == 0
    return out


def main() -> None:
    ref = RefLib()
    for name, fn in (("half", half_vectors), ("store", store_vectors), ("prune", prune_vectors),
                     ("adam", adam_vectors), ("step", step_vectors)):
        data = fn(ref)
        np.savez_compressed(OUT / f"{name}.npz", **data)
        print(name, sum(v.nbytes for v in data.values()), "bytes raw")


if __name__ == "__main__":
    main()
