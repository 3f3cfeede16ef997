"""One rank of the data-parallel GPU parity test (launched by
tests/test_gpu_dp.py through torch.distributed.run).  Builds a small model,
steps it with rank-specific dense gradients through libsamo_cuda.so (NCCL
exchange, bucketed and overlapped unless SAMO_OVERLAP=0) and saves the final
state for the parent to check against the oracle."""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Oracle  # noqa: E402  (test infrastructure: inputs only)
from paper_2302_05045_b200 import dist as sdist  # noqa: E402
from paper_2302_05045_b200 import samo  # noqa: E402

DENSE_LEN = [40000, 3000, 100003, 512]
PRUNABLE = [True, True, True, False]
STEPS = int(os.environ.get("SAMO_DP_STEPS", "4"))  # the stress variant runs 40
INF_STEP, INF_RANK = 2, 1
BF16 = os.environ.get("SAMO_DP_BF16") == "1"  # bfloat16 dense gradients


def decode(o: Oracle, h):
    """The oracle's widening of the dense gradient type."""
    return o.bf16_to_float(h) if BF16 else o.h2f(h)


def inputs(o: Oracle, world: int):
    rng = np.random.default_rng(0)
    vals = [(rng.standard_normal(d) * 0.05).astype(np.float32) for d in DENSE_LEN]
    sets = o.magnitude_prune(vals, PRUNABLE, 0.9)
    grads = {}
    for rank in range(world):
        for s in range(STEPS):
            for l, d in enumerate(DENSE_LEN):
                h = o.synth_f16(0, d, sdist.rank_seed(11, rank), 100 * s + l, 2.0**-7, 1024.0)
                if BF16:  # the same values as bfloat16 patterns (truncated), wider exponents mixed in
                    h = (o.h2f(h).view(np.uint32) >> 16).astype(np.uint16)
                    h[::97] = (h[::97] & np.uint16(0x807F)) | np.uint16(0x4700)  # ~ 2^15 .. 2^16
                if s == INF_STEP and rank == INF_RANK and l == 2:
                    h[int(sets[2][5])] = 0x7F80 if BF16 else 0x7C00
                grads[(rank, s, l)] = h
    return vals, sets, grads


def main() -> None:
    out_dir = Path(sys.argv[1])
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    o = Oracle()
    vals, sets, grads = inputs(o, world)
    psets = [samo.PrunedIndexSet(f"l{l}", d, torch.from_numpy(s.view(np.int32)).cuda())
             for l, (d, s) in enumerate(zip(DENSE_LEN, sets))]
    model = samo.SamoModel.from_index_sets(psets, [(d,) for d in DENSE_LEN], tile_elems=1024)
    for l, v in enumerate(vals):
        model.init_layer(l, torch.from_numpy(v).cuda())
    model.set_config(samo.OptimizerConfig(learning_rate=1e-2))
    if BF16:
        model.set_grad_dtype(torch.bfloat16)
    comm = sdist.make_communicator()
    model.attach_comm(comm)
    mode = os.environ.get("SAMO_DP_MODE", "sharded")
    model.set_exchange({"sharded": model.EXCHANGE_SHARDED, "p2p": model.EXCHANGE_P2P,
                        "allreduce": model.EXCHANGE_ALLREDUCE}[mode])
    sink = os.environ.get("SAMO_DP_SINK") == "1"
    # NCCL exchanges at G > 2: keep every step's exchanged fp32 gradient (the
    # arena after the step: replicated for allreduce, the rank's shard for
    # sharded) so the parent can bound the NCCL sum and replay the update.
    save_g = os.environ.get("SAMO_DP_SAVE_G") == "1"
    gsum = {}
    for s in range(STEPS):
        g = [torch.from_numpy(grads[(rank, s, l)].view(np.int16)).cuda() for l in range(len(DENSE_LEN))]
        if sink:  # per-layer backward sinks (last layer first), then exchange + update
            for l in reversed(range(len(DENSE_LEN))):
                model.sink_dense(l, g[l])
            model.step_sunk()
        else:
            model.set_grads(g)
            model.step(graph=os.environ.get("SAMO_DP_GRAPH") == "1")
        if save_g:
            for l in range(len(DENSE_LEN)):
                gsum[f"g32_{s}_{l}"] = model.read(l, "grad32").cpu().numpy()
    torch.cuda.synchronize()
    rec = model.step_record()
    ranges = np.array(model.shard_ranges(), np.uint64).reshape(-1, 2)
    out = {"t": np.array([rec.t]), "skipped": np.array([rec.skipped_steps]),
           "norm": np.array([rec.grad_norm], np.float32), "shard": ranges,
           "k_off": np.array([model.view(l).k_offset for l in range(len(DENSE_LEN))], np.uint64)}
    out.update(gsum)
    for l in range(len(DENSE_LEN)):
        for k in ("theta32", "adam_m", "adam_v"):
            out[f"{k}{l}"] = model.read(l, k).cpu().numpy()
        out[f"theta16_{l}"] = model.read(l, "theta16").cpu().numpy().view(np.uint16)
    np.savez(out_dir / f"dp_rank{rank}.npz", **out)
    model.close()
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
