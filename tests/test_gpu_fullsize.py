"""GPU: the headline configuration (GPT-2.7B set, p = 0.9, 388 tensors,
2.65e9 parameters) and BASELINE config 3 (GPT-1.3B set, p = 0.8 / 0.95, 292
tensors) at full size, EVERY tensor compared bit for bit with the oracle:

* K0: every layer's kept index set equals the oracle's magnitude_prune
  (prune.hpp:99-170, per-layer scope) on the same synthetic weights;
* four device steps through the production single-GPU step (K123, eager then
  graph): two finite steps, a step whose gradients hold +inf at one kept
  element of one layer (global skip, train.hpp:632-639 -> K123's speculative
  buffers are dropped and the skip-repair kernel restores theta16), then one
  more finite step;
* after them every layer's theta32 / adam_m / adam_v / theta16 equals the
  oracle's optimizer_step (train.hpp:617-656) replayed on that layer, bit for
  bit; the oracle runs one layer per host thread (ctypes releases the GIL);
* check_state_invariants over the whole model, step counters (t = 3,
  skipped = 1), and the recorded grad norm of step 1 against an independent
  fp64 norm of all kept gradients (rel 1e-5).
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

SEED = 3
F16_INF = 0x7C00


def _bits32(t):
    return t.cpu().numpy().view(np.uint32)


def _grad_sid(step: int, layer: int) -> int:
    return 100 * step + layer


def _oracle_layer(oracle, i, n, prunable, bound, sparsity, dev, steps, skip_step):
    """Replays layer i on the CPU oracle; returns the names of mismatches."""
    from oracle.oracle import Cfg, StepState
    vals = oracle.synth_f32(0, n, SEED, 2 * i, bound)
    idx = oracle.magnitude_prune([vals], [prunable], sparsity)[0]
    bad = []
    if not np.array_equal(dev["idx"], idx):
        return ["mask"]
    theta = oracle.compress(vals, idx)
    del vals
    m, v, g32 = (np.zeros_like(theta) for _ in range(3))
    t16 = [np.zeros(n, np.uint16)]
    cfg, st = Cfg(), StepState()
    for s in range(steps):
        gh = oracle.synth_f16(0, n, SEED + 1, _grad_sid(s, i), 2.0**-7, 1024.0)
        if s == skip_step:
            if idx.size == 0:
                continue  # an empty layer sees no gradient; the global skip leaves it as is
            gh[idx[0]] = F16_INF  # every layer skips, as the global flag makes the device do
        oracle.optimizer_step([n], [idx.size], idx, [gh], theta, m, v, g32, t16, cfg, st)
    if idx.size and (st.t, st.skipped) != (steps - 1, 1):
        bad.append("counters")
    for name, want in (("theta32", theta.view(np.uint32)), ("adam_m", m.view(np.uint32)),
                       ("adam_v", v.view(np.uint32)), ("theta16", t16[0])):
        if not np.array_equal(dev[name], want):
            bad.append(name)
    return bad


@pytest.mark.parametrize("name,p", [("gpt-2.7b", 0.9), ("gpt-1.3b", 0.8), ("gpt-1.3b", 0.95)])
def test_gpt_fullsize_every_tensor(cuda, oracle, name, p):
    from paper_2302_05045_b200 import samo, workloads
    wl = workloads.get(name, p)
    assert len(wl.tensors) == {"gpt-2.7b": 388, "gpt-1.3b": 292}[name]
    vals = [samo.synth_uniform_f32(t.numel, SEED, 2 * i, t.init_bound) for i, t in enumerate(wl.tensors)]
    sets = samo.magnitude_prune([samo.LayerParams(t.name, v, t.prunable) for t, v in zip(wl.tensors, vals)],
                                wl.sparsity)
    for t, s in zip(wl.tensors, sets):
        want = oracle.unpruned_count(wl.sparsity, t.numel) if t.prunable else t.numel
        assert s.count() == want, t.name
    model = samo.SamoModel.from_index_sets(sets, [t.shape for t in wl.tensors], 0)
    for l, v in enumerate(vals):
        model.init_layer(l, v)
    model.set_config(samo.OptimizerConfig())
    del vals
    torch.cuda.empty_cache()

    steps, skip_step, inf_layer = 4, 2, len(wl.tensors) // 2
    kept_sq = torch.zeros((), dtype=torch.float64, device="cuda")
    for s in range(steps):
        grads = [samo.synth_uniform_f16(t.numel, SEED + 1, _grad_sid(s, i), 2.0**-7, 1024.0)
                 for i, t in enumerate(wl.tensors)]
        if s == skip_step:
            k = int(sets[inf_layer].as_int64()[0])
            grads[inf_layer].view(torch.int16)[k] = F16_INF
        model.set_grads(grads)
        model.step(graph=(s >= 1))
        if s == 1:  # independent fp64 norm of the unscaled kept gradients
            for i in range(len(wl.tensors)):
                g = grads[i][sets[i].as_int64()].double() / 1024.0
                kept_sq += (g * g).sum()
            torch.cuda.synchronize()
            rec = model.step_record()
            exact = float(kept_sq.sqrt())
            assert abs(rec.grad_norm - exact) <= 1e-5 * exact
        del grads
    torch.cuda.synchronize()
    model.check_invariants()
    rec = model.step_record()
    assert rec.t == steps - 1 and rec.skipped_steps == 1

    workers = max(1, min(32, os.cpu_count() or 1))
    failures, pending = [], []
    with ThreadPoolExecutor(workers) as pool:
        for i, t in enumerate(wl.tensors):
            dev = {"idx": sets[i].indices.cpu().numpy().view(np.uint32),
                   "theta32": _bits32(model.read(i, "theta32")),
                   "adam_m": _bits32(model.read(i, "adam_m")),
                   "adam_v": _bits32(model.read(i, "adam_v")),
                   "theta16": model.read(i, "theta16").reshape(-1).cpu().numpy().view(np.uint16)}
            pending.append((t.name, pool.submit(_oracle_layer, oracle, i, t.numel, t.prunable,
                                                t.init_bound, wl.sparsity, dev, steps, skip_step)))
            while len(pending) > 2 * workers:  # bound the host copies in flight
                nm, f = pending.pop(0)
                failures += [f"{nm}:{b}" for b in f.result()]
        for nm, f in pending:
            failures += [f"{nm}:{b}" for b in f.result()]
    model.close()
    assert not failures, failures[:20]


def test_max_layer_size(cuda, oracle):
    """The largest layer the reference allows (dense_len < 2^32, prune.hpp:
    106-109): 32-bit tile offsets, K0's histograms and the step kernels at
    the edge.  K0 count and top-|v| property, two steps, whole-layer
    invariants (theta16 == expand(half(theta32)), zeros elsewhere) and the
    kept elements bit-exact vs the oracle's optimizer_step arithmetic."""
    from paper_2302_05045_b200 import samo
    from oracle.oracle import Cfg
    n = 2**32 - 64
    if torch.cuda.mem_get_info()[0] < 64e9:
        pytest.skip("needs ~64 GB of free device memory")
    p = 0.9999
    w = samo.synth_uniform_f32(n, 5, 0, 0.05)
    sets = samo.magnitude_prune([samo.LayerParams("big", w, True)], p)
    keep = oracle.unpruned_count(p, n)
    assert sets[0].count() == keep
    idx_t = sets[0].as_int64()  # uint32 indices held in an int32 tensor
    idx = sets[0].indices.cpu().numpy().view(np.uint32)
    assert np.all(np.diff(idx.astype(np.int64)) > 0) and int(idx[-1]) < n
    thr = w[idx_t].abs().min()
    assert int((w.abs() > thr).sum()) <= keep  # nothing larger was dropped
    model = samo.SamoModel.from_index_sets(sets, [(n,)], 0)
    model.init_layer(0, w)
    theta = w[idx_t].cpu().numpy()
    del w
    torch.cuda.empty_cache()
    model.set_config(samo.OptimizerConfig(learning_rate=1e-2))
    m, v = np.zeros_like(theta), np.zeros_like(theta)
    cfg = Cfg(lr=1e-2)
    b1p = b2p = np.float32(1.0)
    for s in range(2):
        g = samo.synth_uniform_f16(n, 6, s, 2.0**-7, 1024.0)
        model.set_grads([g])
        model.step()
        gk = oracle.h2f(g[idx_t].cpu().numpy().view(np.uint16))
        g32 = (gk * np.float32(1.0 / 1024.0)).astype(np.float32)  # train.hpp:619-624
        b1p, b2p = np.float32(b1p * np.float32(0.9)), np.float32(b2p * np.float32(0.999))
        oracle.adam_update(theta, m, v, g32, cfg, float(np.float32(1) - b1p), float(np.float32(1) - b2p))
        del g
    torch.cuda.synchronize()
    model.check_invariants()
    assert np.array_equal(model.read(0, "theta32").cpu().numpy().view(np.uint32), theta.view(np.uint32))
    assert np.array_equal(model.read(0, "adam_v").cpu().numpy().view(np.uint32), v.view(np.uint32))
    assert model.step_record().t == 2
    model.close()
