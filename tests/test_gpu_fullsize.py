"""GPU: the headline configuration at full size (GPT-2.7B set, p = 0.9, 388
tensors, 2.65e9 parameters), through size-independent properties and
sampled bit-exact layers (the oracle cannot run the whole model in a test):

* K0: every layer keeps exactly unpruned_count(p, n) indices (prune.hpp:76-79),
  non-prunable layers keep all; sampled layers equal the oracle's mask;
* two full device steps, then check_state_invariants over the whole model
  (theta16 == expand(half(theta32)), zeros at every pruned position);
* sampled layers (smallest, an attention projection, an MLP matrix) equal the
  oracle's optimizer_step bit for bit after both steps;
* the recorded grad norm equals an independent fp64 norm of all 2.66e8
  kept gradients (rel 1e-5).
"""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

SEED = 3


def _bits32(t):
    return t.cpu().numpy().view(np.uint32)


def test_gpt_2_7b_fullsize(cuda, oracle):
    from paper_2302_05045_b200 import samo, workloads
    from oracle.oracle import Cfg, StepState
    wl = workloads.get("gpt-2.7b", 0.9)
    assert len(wl.tensors) == 388
    vals = [samo.synth_uniform_f32(t.numel, SEED, 2 * i, t.init_bound) for i, t in enumerate(wl.tensors)]
    sets = samo.magnitude_prune([samo.LayerParams(t.name, v, t.prunable) for t, v in zip(wl.tensors, vals)],
                                wl.sparsity)
    for t, s in zip(wl.tensors, sets):
        want = oracle.unpruned_count(wl.sparsity, t.numel) if t.prunable else t.numel
        assert s.count() == want, t.name
    # sampled layers: the smallest, an attention projection, an MLP matrix
    numel = [t.numel for t in wl.tensors]
    small = int(np.argmin(numel))
    attn = next(i for i, t in enumerate(wl.tensors) if t.prunable and t.shape == (2560, 2560))
    mlp = next(i for i, t in enumerate(wl.tensors) if t.prunable and t.shape == (2560, 10240))
    sample = [small, attn, mlp]
    host_vals = {i: vals[i].cpu().numpy() for i in sample}
    for i in sample:
        want = oracle.magnitude_prune([host_vals[i]], [wl.tensors[i].prunable], wl.sparsity)[0]
        assert np.array_equal(sets[i].indices.cpu().numpy().view(np.uint32), want), wl.tensors[i].name

    model = samo.SamoModel.from_index_sets(sets, [t.shape for t in wl.tensors], 0)
    for l, v in enumerate(vals):
        model.init_layer(l, v)
    model.set_config(samo.OptimizerConfig())
    del vals
    torch.cuda.empty_cache()

    grads = [None] * len(wl.tensors)
    kept_sq = torch.zeros((), dtype=torch.float64, device="cuda")
    for s in range(2):
        for i, t in enumerate(wl.tensors):
            grads[i] = samo.synth_uniform_f16(t.numel, SEED + 1, 100 * s + i, 2.0**-7, 1024.0)
        model.set_grads(grads)
        model.step(graph=(s == 1))
        if s == 1:  # independent fp64 norm of the unscaled kept gradients
            for i in range(len(wl.tensors)):
                g = grads[i][sets[i].indices.long()].double() / 1024.0
                kept_sq += (g * g).sum()
    torch.cuda.synchronize()
    model.check_invariants()
    rec = model.step_record()
    assert rec.t == 2 and rec.skipped_steps == 0
    exact = float(kept_sq.sqrt())
    assert abs(rec.grad_norm - exact) <= 1e-5 * exact

    cfg, st = Cfg(), StepState()
    for i in sample:
        idx = sets[i].indices.cpu().numpy().view(np.uint32)
        n = wl.tensors[i].numel
        theta = oracle.compress(host_vals[i], idx)
        m, v, g32 = (np.zeros_like(theta) for _ in range(3))
        t16 = [np.zeros(n, np.uint16)]
        st = StepState()
        for s in range(2):
            gh = oracle.synth_f16(0, n, SEED + 1, 100 * s + i, 2.0**-7, 1024.0)
            oracle.optimizer_step([n], [idx.size], idx, [gh], theta, m, v, g32, t16, cfg, st)
        name = wl.tensors[i].name
        assert np.array_equal(_bits32(model.read(i, "theta32")), theta.view(np.uint32)), name
        assert np.array_equal(_bits32(model.read(i, "adam_m")), m.view(np.uint32)), name
        assert np.array_equal(_bits32(model.read(i, "adam_v")), v.view(np.uint32)), name
        assert np.array_equal(model.read(i, "theta16").reshape(-1).cpu().numpy().view(np.uint16), t16[0]), name
    model.close()


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
