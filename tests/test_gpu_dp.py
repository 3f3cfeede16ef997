"""Data-parallel parity on >= 2 GPUs: the NCCL exchange of the compressed
gradient arena, bucketed and overlapped with the step kernels.

Tolerance: none at G = 2 — a two-operand fp32 sum is order-independent, so
every replica must equal the oracle (rank-ascending fp32 sum, then the
reference's Adam / downcast / expand) bit for bit, including the step skipped
because one rank saw +inf.  Skipped when fewer than two GPUs are visible."""
from __future__ import annotations

import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

HERE = Path(__file__).resolve().parent


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _expected(oracle, world, steps=4):
    sys.path.insert(0, str(HERE))
    os.environ["SAMO_DP_STEPS"] = str(steps)
    import importlib
    import dp_worker as W
    W = importlib.reload(W)
    from oracle.oracle import Cfg
    vals, sets, grads = W.inputs(oracle, world)
    L = len(W.DENSE_LEN)
    theta = [oracle.compress(v, s) for v, s in zip(vals, sets)]
    m = [np.zeros_like(t) for t in theta]
    v = [np.zeros_like(t) for t in theta]
    cfg = Cfg(lr=1e-2)
    b1p = b2p = np.float32(1.0)
    t = skipped = 0
    inv = np.float32(1.0) / np.float32(1024.0) * (np.float32(1.0) / np.float32(world))
    for s in range(W.STEPS):
        g = []
        for l in range(L):
            per_rank = [(W.decode(oracle, oracle.compress(grads[(r, s, l)], sets[l])) * inv).astype(np.float32)
                        for r in range(world)]
            g.append(oracle.dp_sum(per_rank)[0])
        if not all(np.all(np.isfinite(x)) for x in g):
            skipped += 1
            continue
        t += 1
        b1p = np.float32(b1p * np.float32(0.9))
        b2p = np.float32(b2p * np.float32(0.999))
        for l in range(L):
            oracle.adam_update(theta[l], m[l], v[l], g[l], cfg, float(np.float32(1) - b1p),
                               float(np.float32(1) - b2p))
    t16 = [oracle.expand(oracle.f2h(theta[l]), sets[l], (W.DENSE_LEN[l],)) for l in range(L)]
    return theta, m, v, t16, t, skipped


def _run(tmp_path, mode, world, steps=4, save_g=False):
    env = dict(os.environ)
    env["SAMO_DP_SAVE_G"] = "1" if save_g else "0"
    env["SAMO_DP_STEPS"] = str(steps)
    env["SAMO_DP_MODE"] = mode.split("-")[0] if mode.split("-")[0] in ("sharded", "p2p") else "allreduce"
    env["SAMO_OVERLAP"] = "0" if mode == "staged" else "1"
    env["SAMO_DP_GRAPH"] = "1" if mode.endswith("graph") else "0"
    env["SAMO_BUCKETS"] = "5"
    # p2p: the pipelined peer-signalled step (5 buckets, some empty on some
    # ranks); p2p-serial: one shard launch between two NCCL barriers.
    env["SAMO_P2P_BUCKETS"] = "1" if mode == "p2p-serial" else "5"
    env["SAMO_DP_SINK"] = "1" if mode == "p2p-sink" else "0"  # per-layer sinks + step_sunk
    env["SAMO_P2P_PUSH"] = "0" if mode == "p2p-pull" else "1"  # the shard update pulls the gradients
    env["SAMO_DP_BF16"] = "1" if mode.endswith("-bf16") else "0"  # bfloat16 dense gradients
    os.environ["SAMO_DP_BF16"] = env["SAMO_DP_BF16"]  # the parent's oracle replay reads it too
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           str(HERE / "dp_worker.py"), str(tmp_path)]
    for _ in range(3):  # a rendezvous port taken between _port() and bind: retry on another
        res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
        if res.returncode == 0 or "EADDRINUSE" not in res.stderr:
            break
        cmd[cmd.index("--master-port") + 1] = str(_port())
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    return [dict(np.load(tmp_path / f"dp_rank{i}.npz")) for i in range(world)]


def _check(r, oracle, world, mode, steps=4):
    theta, m, v, t16, t, skipped = _expected(oracle, world, steps)
    covered = 0
    for rr in r:
        assert int(rr["t"][0]) == t and int(rr["skipped"][0]) == skipped == 1
        for l in range(len(theta)):
            # theta16 is complete on every rank; theta32/m/v are authoritative
            # in the rank's shard (everything unless the exchange is sharded)
            assert np.array_equal(rr[f"theta16_{l}"], t16[l]), l
        for k0, k1 in (tuple(int(x) for x in row) for row in rr["shard"]):
            for l in range(len(theta)):
                off = int(rr["k_off"][l])
                lo, hi = max(k0 - off, 0), min(k1 - off, len(theta[l]))
                if hi <= lo:
                    continue
                covered += hi - lo
                for name, want in (("theta32", theta), ("adam_m", m), ("adam_v", v)):
                    got = rr[f"{name}{l}"][lo:hi].view(np.uint32)
                    assert np.array_equal(got, want[l][lo:hi].view(np.uint32)), (name, l)
    n = sum(len(x) for x in theta)
    assert covered == (n if mode.split("-")[0] in ("sharded", "p2p") else world * n)


@pytest.mark.parametrize("mode", ["p2p", "p2p-serial", "p2p-graph", "p2p-sink", "p2p-pull",
                                  "sharded", "sharded-graph", "overlap",
                                  "staged", "graph", "p2p-bf16", "sharded-bf16", "overlap-bf16"])
def test_dp_two_gpus_bit_exact(tmp_path, oracle, mode):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    _check(_run(tmp_path, mode, 2), oracle, 2, mode)


@pytest.mark.parametrize("mode", ["p2p", "p2p-serial", "p2p-graph", "p2p-sink", "p2p-pull", "p2p-bf16"])
def test_dp_four_gpus_p2p_bit_exact(tmp_path, oracle, mode):
    """The fused exchange sums in rank order: bit-exact for G = 4 too."""
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    _check(_run(tmp_path, mode, 4), oracle, 4, mode)


def test_dp_three_gpus_p2p_bit_exact(tmp_path, oracle):
    """Non-power-of-two G: 1/G is inexact, but the kernel applies the same
    fp32 scale (1/loss_scale * 1/G) per rank before the rank-ordered sum as
    the oracle, so replicas still match it bit for bit."""
    if torch.cuda.device_count() < 3:
        pytest.skip("needs 3 GPUs")
    _check(_run(tmp_path, "p2p", 3), oracle, 3, "p2p")


def test_dp_four_gpus_p2p_stress(tmp_path, oracle):
    """40 pipelined push-mode steps: the peer-signal epochs wrap through many
    steps and every replica must still equal the oracle bit for bit."""
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    _check(_run(tmp_path, "p2p", 4, steps=40), oracle, 4, "p2p", steps=40)


def _check_nccl_tolerance(r, oracle, world, mode, steps=4):
    """Parity of an NCCL exchange whose summation order NCCL defines (ring
    chunks, or NVLS reductions in the switch), at any G:

    1. exchange: every exchanged fp32 gradient element g (every step, the
       authoritative ranges of every rank) satisfies
           |g - S| <= (G-1) * 2^-24 * sum_r |g_r|
       against the exact sum S of the ranks' unscaled gradients (fp64, exact
       for these inputs), the bound for fp32 summation of G terms in any
       order; non-finite elements sit exactly where S is non-finite, and
       allreduce replicas are bit-identical to each other;
    2. update: the oracle's Adam / downcast / expand replayed on the device's
       own exchanged gradients equals the device theta32 / m / v / theta16
       bit for bit (only the summation order is NCCL's);
    3. end to end: theta32 against the oracle that sums rank-ascending is
       within 1e-6 relative, plus the first-order Adam sensitivity
       4 * lr * sum_s bound_s / |S_s| where a sum cancels."""
    import dp_worker as W
    from oracle.oracle import Cfg
    theta_o, _, _, _, t_o, skipped_o = _expected(oracle, world, steps)
    vals, sets, grads = W.inputs(oracle, world)
    L = len(W.DENSE_LEN)
    cfg = Cfg(lr=1e-2)
    inv = np.float32(1.0) / np.float32(1024.0) * (np.float32(1.0) / np.float32(world))
    theta = [oracle.compress(v, s) for v, s in zip(vals, sets)]
    m = [np.zeros_like(t) for t in theta]
    v = [np.zeros_like(t) for t in theta]
    sens = [np.zeros(len(t)) for t in theta]
    b1p = b2p = np.float32(1.0)
    t = skipped = 0
    worst = 0.0
    replicated = mode.split("-")[0] not in ("sharded", "p2p")
    for s in range(steps):
        g, gb = [], []
        for l in range(L):
            per_rank = [(W.decode(oracle, oracle.compress(grads[(q, s, l)], sets[l])) * inv).astype(np.float32)
                        for q in range(world)]
            stack = np.stack(per_rank).astype(np.float64)
            exact = stack.sum(axis=0)
            bound = (world - 1) * 2.0**-24 * np.abs(stack).sum(axis=0)
            n_l = len(theta[l])
            got = np.zeros(n_l, np.float32)
            seen = np.zeros(n_l, bool)
            for rr in r:
                off = int(rr["k_off"][l])
                for k0, k1 in (tuple(int(x) for x in row) for row in rr["shard"]):
                    lo, hi = max(k0 - off, 0), min(k1 - off, n_l)
                    if hi <= lo:
                        continue
                    part = rr[f"g32_{s}_{l}"][lo:hi]
                    if replicated and seen[lo:hi].any():
                        assert np.array_equal(part.view(np.uint32), got[lo:hi].view(np.uint32)), \
                            ("replicas differ", s, l)
                    got[lo:hi] = part
                    seen[lo:hi] = True
            assert seen.all(), (s, l)
            fin = np.isfinite(exact)
            assert np.array_equal(np.isfinite(got), fin), (s, l)
            err = np.abs(got[fin].astype(np.float64) - exact[fin])
            assert np.all(err <= bound[fin] * (1 + 2.0**-20)), (s, l, float((err - bound[fin]).max()))
            nz = fin & (bound > 0)
            if nz.any():
                worst = max(worst, float((err[nz[fin]] / bound[nz]).max()))
            g.append(got)
            gb.append((exact, bound))
        if not all(np.all(np.isfinite(x)) for x in g):
            skipped += 1
            continue
        for l, (exact, bound) in enumerate(gb):
            with np.errstate(divide="ignore", invalid="ignore"):
                sens[l] += np.where(np.abs(exact) > 0, bound / np.abs(exact), np.inf)
        t += 1
        b1p = np.float32(b1p * np.float32(0.9))
        b2p = np.float32(b2p * np.float32(0.999))
        for l in range(L):
            oracle.adam_update(theta[l], m[l], v[l], g[l], cfg, float(np.float32(1) - b1p),
                               float(np.float32(1) - b2p))
    assert (t, skipped) == (t_o, skipped_o)
    t16 = [oracle.expand(oracle.f2h(theta[l]), sets[l], (W.DENSE_LEN[l],)) for l in range(L)]
    for rr in r:
        assert int(rr["t"][0]) == t and int(rr["skipped"][0]) == skipped
        for l in range(L):
            assert np.array_equal(rr[f"theta16_{l}"], t16[l]), l
        for k0, k1 in (tuple(int(x) for x in row) for row in rr["shard"]):
            for l in range(L):
                off = int(rr["k_off"][l])
                lo, hi = max(k0 - off, 0), min(k1 - off, len(theta[l]))
                if hi <= lo:
                    continue
                for name, want in (("theta32", theta), ("adam_m", m), ("adam_v", v)):
                    got = rr[f"{name}{l}"][lo:hi].view(np.uint32)
                    assert np.array_equal(got, want[l][lo:hi].view(np.uint32)), (name, l)
    rel = 0.0
    for l in range(L):
        d = np.abs(theta[l].astype(np.float64) - theta_o[l].astype(np.float64))
        tol = 1e-6 * np.abs(theta_o[l].astype(np.float64)) + 4 * cfg.lr * sens[l]
        assert np.all(d <= tol), (l, float((d - tol).max()))
        rel = max(rel, float((d / np.maximum(np.abs(theta_o[l]), 1e-30)).max()))
    print(f"{mode} G={world}: max |g - S| / bound = {worst:.3f}; max theta32 rel vs rank-ascending "
          f"oracle = {rel:.2e}")


@pytest.mark.parametrize("G", [3, 4])
@pytest.mark.parametrize("mode", ["overlap", "staged", "graph", "sharded", "sharded-graph"])
def test_dp_nccl_tolerance(tmp_path, oracle, mode, G):
    """The north-star exchange (NCCL allreduce of the compressed fp32 arena,
    and the NCCL reduce-scatter / all-gather sharded form) at G = 3 and 4,
    where the NCCL summation order differs from the oracle's rank-ascending
    sum: tolerance on the sum, bit-exact downstream (_check_nccl_tolerance)."""
    if torch.cuda.device_count() < G:
        pytest.skip(f"needs {G} GPUs")
    _check_nccl_tolerance(_run(tmp_path, mode, G, save_g=True), oracle, G, mode)


def test_dp_nccl_tolerance_two_gpus(tmp_path, oracle):
    """G = 2 through the same checker (bit-exact there anyway)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    _check_nccl_tolerance(_run(tmp_path, "overlap", 2, save_g=True), oracle, 2, "overlap")


def _local_group_run(oracle, G, steps=4, sink=False, devices=None):
    """G models on cuda:0 as the ranks of one peer-to-peer group
    (samo_model_attach_local_group + samo_local_group_step): the same inputs
    and outputs as dp_worker.py.  devices: model r on cuda:devices[r] (a
    group across GPUs in one process)."""
    sys.path.insert(0, str(HERE))
    os.environ["SAMO_DP_STEPS"] = str(steps)
    import importlib
    import dp_worker as W
    W = importlib.reload(W)
    from paper_2302_05045_b200 import samo
    vals, sets, grads = W.inputs(oracle, G)
    L = len(W.DENSE_LEN)
    models = []
    for r in range(G):
        if devices:
            torch.cuda.set_device(devices[r])
        psets = [samo.PrunedIndexSet(f"l{l}", d, torch.from_numpy(s.view(np.int32)).cuda())
                 for l, (d, s) in enumerate(zip(W.DENSE_LEN, sets))]
        m = samo.SamoModel.from_index_sets(psets, [(d,) for d in W.DENSE_LEN], tile_elems=1024)
        for l, v in enumerate(vals):
            m.init_layer(l, torch.from_numpy(v).cuda())
        m.set_config(samo.OptimizerConfig(learning_rate=1e-2))
        if W.BF16:
            m.set_grad_dtype(torch.bfloat16)
        models.append(m)
    if devices:
        torch.cuda.set_device(devices[0])
        for r in range(G):
            torch.cuda.synchronize(devices[r])
    samo.SamoModel.attach_local_group(models)
    dev = {(r, s): [torch.from_numpy(grads[(r, s, l)].view(np.int16)).cuda(devices[r] if devices else None)
                    for l in range(L)]
           for r in range(G) for s in range(W.STEPS)}
    torch.cuda.synchronize()
    for s in range(W.STEPS):
        if sink:  # per-layer backward sinks, last layer first, pushed to the owners
            for r in range(G):
                for l in reversed(range(L)):
                    models[r].sink_dense(l, dev[(r, s)][l])
            samo.SamoModel.local_group_step_sunk(models)
        else:
            for r in range(G):
                models[r].set_grads(dev[(r, s)])
            samo.SamoModel.local_group_step(models)
    torch.cuda.synchronize()
    out = []
    for m in models:
        rec = m.step_record()
        rr = {"t": np.array([rec.t]), "skipped": np.array([rec.skipped_steps]),
              "shard": np.array(m.shard_ranges(), np.uint64).reshape(-1, 2),
              "k_off": np.array([m.view(l).k_offset for l in range(L)], np.uint64)}
        for l in range(L):
            for k in ("theta32", "adam_m", "adam_v"):
                rr[f"{k}{l}"] = m.read(l, k).cpu().numpy()
            rr[f"theta16_{l}"] = m.read(l, "theta16").cpu().numpy().view(np.uint16)
        out.append(rr)
    for m in models:
        m.close()
    return out


@pytest.mark.parametrize("G,env", [(3, {}), (5, {}), (8, {}), (8, {"SAMO_P2P_PUSH": "0"}),
                                   (2, {"SAMO_P2P_BUCKETS": "5"}), (7, {"SAMO_P2P_BUCKETS": "3"}),
                                   (3, {"SAMO_DP_BF16": "1"}), (8, {"SAMO_DP_BF16": "1", "SAMO_P2P_PUSH": "0"})],
                         ids=lambda x: str(x) if isinstance(x, int) else "-".join(f"{k[9:]}{v}" for k, v in x.items()) or "default")
def test_local_group_p2p_bit_exact(cuda, oracle, monkeypatch, G, env):
    """The pipelined peer-to-peer step at G up to 8 on ONE GPU: G models on
    cuda:0 are the ranks (peers mapped directly, no NCCL), stepped phase by
    phase on one stream.  The same kernels, peer stores, signals and bucket
    plans as across GPUs, so every replica must equal the oracle bit for bit
    — including G = 5, 7, 8, which the pool's 2- and 4-GPU boxes cannot run
    as processes."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _check(_local_group_run(oracle, G), oracle, G, "p2p")


@pytest.mark.parametrize("G", [2, 4, 8])
def test_local_group_push_sinks_bit_exact(cuda, oracle, monkeypatch, G):
    """The exchange sent during the backward: each rank's per-layer sinks
    (last layer first, train.hpp:287-313) push the layer's kept binary16
    gradients straight into their owners' receive buffers; the step after
    them is only the flag exchange, the shard updates and the expand.  Every
    replica equals the oracle bit for bit."""
    if G == 2:  # a local group runs the pipelined schedule (one bucket is the G = 2 default)
        monkeypatch.setenv("SAMO_P2P_BUCKETS", "5")
    _check(_local_group_run(oracle, G, sink=True), oracle, G, "p2p")


def test_local_group_push_dw_sinks_equal_dense_sinks(cuda):
    """Fused dW sinks in push mode (the epilogue gathers into scratch, a copy
    pushes to the owners) give the same state as dense sinks of the same dW
    (samo_dw_gemm_f16), at G = 4 over three steps."""
    from paper_2302_05045_b200 import samo
    G, batch = 4, 64
    shapes = [(64, 128), (256, 32), (8, 8)]
    rng = np.random.default_rng(3)
    vals = [torch.from_numpy((rng.standard_normal(a * b) * 0.05).astype(np.float32)).cuda() for a, b in shapes]
    sets = samo.magnitude_prune([samo.LayerParams(f"l{i}", v, True) for i, v in enumerate(vals)], 0.7)

    def group():
        ms = []
        for _ in range(G):
            m = samo.SamoModel.from_index_sets(sets, shapes, tile_elems=1024)
            for l, v in enumerate(vals):
                m.init_layer(l, v)
            m.set_config(samo.OptimizerConfig(learning_rate=1e-2))
            ms.append(m)
        samo.SamoModel.attach_local_group(ms)
        return ms
    fused, dense = group(), group()
    for s in range(3):
        xs = {(r, l): torch.from_numpy((rng.standard_normal((batch, a)) * 0.5).astype(np.float16)).cuda()
              for r in range(G) for l, (a, b) in enumerate(shapes)}
        dys = {(r, l): torch.from_numpy((rng.standard_normal((batch, b)) * 8.0).astype(np.float16)).cuda()
               for r in range(G) for l, (a, b) in enumerate(shapes)}
        for r in range(G):
            for l in reversed(range(len(shapes))):
                fused[r].sink_dw(l, xs[(r, l)], dys[(r, l)])
                dense[r].sink_dense(l, samo.dw_gemm(xs[(r, l)], dys[(r, l)]).reshape(-1))
        samo.SamoModel.local_group_step_sunk(fused)
        samo.SamoModel.local_group_step_sunk(dense)
    torch.cuda.synchronize()
    for r in range(G):
        assert fused[r].step_record().t == dense[r].step_record().t == 3
        for l in range(len(shapes)):
            for k in ("theta32", "adam_v", "theta16"):
                assert torch.equal(fused[r].read(l, k).view(torch.int16 if k == "theta16" else torch.int32),
                                   dense[r].read(l, k).view(torch.int16 if k == "theta16" else torch.int32)), (r, l, k)
    for m in fused + dense:
        m.close()


def test_local_group_across_devices_bit_exact(cuda, oracle, monkeypatch):
    """One process, one model per GPU, peers mapped directly (the harness
    the NVLink profile uses, tools/nvlink_group_ncu.py): every phase of a
    rank runs on its own device, the kernels move the gradients and weights
    over NVLink, and every replica equals the oracle bit for bit."""
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs 2 GPUs")
    G = min(n, 4)
    monkeypatch.setenv("SAMO_P2P_BUCKETS", "5")
    _check(_local_group_run(oracle, G, devices=list(range(G))), oracle, G, "p2p")


def test_local_group_eight_ranks_stress(cuda, oracle):
    """40 steps of an 8-rank local group: the signal epochs advance through
    many steps and every replica still equals the oracle bit for bit."""
    _check(_local_group_run(oracle, 8, steps=40), oracle, 8, "p2p", steps=40)


def test_local_group_member_step_is_refused(cuda):
    """A local group's ranks share one host thread: stepping one member on
    its own would wait for the others forever, so it fails at once."""
    from paper_2302_05045_b200 import samo
    idx = torch.arange(0, 4096, 3, dtype=torch.int32, device="cuda")
    models = [samo.SamoModel.from_index_sets([samo.PrunedIndexSet("w", 4096, idx)], [(4096,)]) for _ in range(3)]
    for m in models:
        m.init_layer(0, torch.zeros(4096, device="cuda"))
    samo.SamoModel.attach_local_group(models)
    g = torch.zeros(4096, dtype=torch.float16, device="cuda")
    for m in models:
        m.set_grads([g])
    with pytest.raises(samo.StateError):
        models[0].step()
    # the same members in another order are not this group (each rank's peer
    # map must be exactly the list passed), nor is a list with a stranger
    with pytest.raises(samo.StateError):
        samo.SamoModel.local_group_step([models[0], models[2], models[1]])
    other = samo.SamoModel.from_index_sets([samo.PrunedIndexSet("w", 4096, idx)], [(4096,)])
    other.init_layer(0, torch.zeros(4096, device="cuda"))
    with pytest.raises(samo.StateError):
        samo.SamoModel.local_group_step([models[0], models[1], other])
    other.close()
    samo.SamoModel.local_group_step(models)  # the group step still works
    torch.cuda.synchronize()
    assert all(m.step_record().t == 1 for m in models)
    for m in models:
        m.close()
