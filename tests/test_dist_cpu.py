"""CPU, world_size 2 over gloo: the host side of the data-parallel path.

* the NCCL unique id reaches every rank unchanged (paper_2302_05045_b200.dist);
* the exchange semantics the CUDA step implements — per-rank compressed
  gradients unscaled with 1/G folded in, one sum over ranks, skip on every
  rank when any rank saw a non-finite gradient — reproduced with the oracle
  and a gloo allreduce, checked bit-exact against the oracle's rank-ordered
  sum (G = 2 sums are order-independent).
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, out_dir: str) -> None:
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        from pathlib import Path
        sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
        from oracle.oracle import Oracle
        from paper_2302_05045_b200 import dist as sdist

        uid = sdist.broadcast_unique_id()
        o = Oracle()
        dense_len = [5000, 300]
        rng = np.random.default_rng(0)  # identical weights/mask on every rank
        vals = [rng.standard_normal(d).astype(np.float32) for d in dense_len]
        sets = o.magnitude_prune(vals, [True, False], 0.9)
        inv = np.float32(1.0) / np.float32(1024.0) * (np.float32(1.0) / np.float32(world))
        flags, sums = [], []
        for step in range(3):
            parts = []
            bad = 0.0
            for l, d in enumerate(dense_len):
                h = o.synth_f16(0, d, sdist.rank_seed(7, rank), 10 * step + l, 2.0**-7, 1024.0)
                if step == 1 and rank == 1 and l == 0:
                    h[int(sets[0][3])] = 0x7C00  # +inf on one rank only
                g = o.h2f(o.compress(h, sets[l])) * inv
                bad += float(not np.all(np.isfinite(g)))
                parts.append(g.astype(np.float32))
            arena = torch.from_numpy(np.concatenate(parts + [np.array([bad], np.float32)]))
            dist.all_reduce(arena, op=dist.ReduceOp.SUM)
            a = arena.numpy()
            sums.append(a[:-1].copy())
            flags.append(float(a[-1]))
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), uid=np.frombuffer(uid, np.uint8),
                 flags=np.array(flags), **{f"sum{s}": v for s, v in enumerate(sums)})
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange_semantics(tmp_path, oracle):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    r = [dict(np.load(tmp_path / f"rank{i}.npz")) for i in range(world)]
    # one unique id everywhere
    assert np.array_equal(r[0]["uid"], r[1]["uid"]) and r[0]["uid"].any()
    # the skip indicator is the same on both ranks and set only on step 1
    assert r[0]["flags"].tolist() == r[1]["flags"].tolist() == [0.0, 1.0, 0.0]
    # bit-identical replicas, equal to the oracle's rank-ordered fp32 sum
    from paper_2302_05045_b200 import dist as sdist
    dense_len = [5000, 300]
    rng = np.random.default_rng(0)
    vals = [rng.standard_normal(d).astype(np.float32) for d in dense_len]
    sets = oracle.magnitude_prune(vals, [True, False], 0.9)
    inv = np.float32(1.0) / np.float32(1024.0) * np.float32(0.5)
    for step in (0, 2):
        per_rank = []
        for rank in range(world):
            parts = []
            for l, d in enumerate(dense_len):
                h = oracle.synth_f16(0, d, sdist.rank_seed(7, rank), 10 * step + l, 2.0**-7, 1024.0)
                parts.append((oracle.h2f(oracle.compress(h, sets[l])) * inv).astype(np.float32))
            per_rank.append(np.concatenate(parts))
        want, _ = oracle.dp_sum(per_rank)
        for i in range(world):
            assert np.array_equal(r[i][f"sum{step}"].view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("G", [2, 4, 8])
def test_power_of_two_folding_is_exact(oracle, G):
    """(sum g_r) * s == sum (g_r * s) for power-of-two s: folding 1/G into the
    unscale changes no bits unless a value underflows."""
    rng = np.random.default_rng(G)
    h = [oracle.synth_f16(0, 4096, 3 + r, 0, 2.0**-7, 1024.0) for r in range(G)]
    g = [oracle.h2f(x) for x in h]
    inv = np.float32(1.0 / 1024.0)
    folded, _ = oracle.dp_sum([(x * (inv * np.float32(1.0 / G))).astype(np.float32) for x in g])
    late, _ = oracle.dp_sum([(x * inv).astype(np.float32) for x in g])
    late = (late * np.float32(1.0 / G)).astype(np.float32)
    assert np.array_equal(folded.view(np.uint32), late.view(np.uint32))
    del rng
