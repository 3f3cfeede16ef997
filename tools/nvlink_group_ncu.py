#!/usr/bin/env python
"""NVLink bytes of the fused P2P kernels, measured (ncu link counters).

One process, one model per GPU (a local group across devices: peers mapped
directly, every phase on the rank's own device), the GPT-2.7B p = 0.9 set;
two warm steps, then the profiled step.  Run under ncu, e.g.

  ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,\\
nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
      -k regex:"k1_gather|k_shard_p2p" --launch-skip <2 warm steps' launches> -c <2 G> \\
      python tools/nvlink_group_ncu.py

Measurement tool only; prints the algorithmic link bytes per rank to compare."""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2302_05045_b200 import samo, workloads  # noqa: E402


def main() -> None:
    os.environ.setdefault("SAMO_P2P_BUCKETS", "5")  # a local group runs the pipelined exchange
    G = min(torch.cuda.device_count(), int(sys.argv[1]) if len(sys.argv) > 1 else 4)
    assert G >= 2, "needs 2 GPUs"
    wl = workloads.get(sys.argv[2] if len(sys.argv) > 2 else "gpt-2.7b", 0.9)
    models, grads = [], []
    for r in range(G):
        torch.cuda.set_device(r)
        vals = [samo.synth_uniform_f32(t.numel, 1234, 2 * i, t.init_bound) for i, t in enumerate(wl.tensors)]
        sets = samo.magnitude_prune([samo.LayerParams(t.name, v, t.prunable) for t, v in zip(wl.tensors, vals)],
                                    wl.sparsity)
        m = samo.SamoModel.from_index_sets(sets, [t.shape for t in wl.tensors], 0)
        for l, v in enumerate(vals):
            m.init_layer(l, v)
        m.set_config(samo.OptimizerConfig())
        del vals, sets
        g = [samo.synth_uniform_f16(t.numel, 1235 + r, 2 * i + 1, 2.0**-7, 1024.0) for i, t in enumerate(wl.tensors)]
        m.set_grads(g)
        models.append(m)
        grads.append(g)
        torch.cuda.synchronize()
    torch.cuda.set_device(0)
    samo.SamoModel.attach_local_group(models)
    for _ in range(3):  # two warm steps, then the profiled one
        samo.SamoModel.local_group_step(models)
    for r in range(G):
        torch.cuda.synchronize(r)
    phi, n, _ = models[0].totals()
    print(json.dumps({"G": G, "workload": wl.name, "phi": phi, "n": n,
                      "algorithmic_per_rank": {
                          "K1_push_tx_bytes": 2 * n * (G - 1) / G,
                          "shard_weight_push_tx_bytes": 2 * n * (G - 1) / G}}), flush=True)
    for m in models:
        m.close()


if __name__ == "__main__":
    main()
