"""BASELINE config 5: compressed vs dense gradient exchange message sizes on
this box's GPUs (torchrun, NCCL, one process per GPU).  For the GPT-2.7B set
at sparsity p the compressed fp32 gradient arena is 4n bytes (n = kept
elements), the dense alternatives 4*phi (fp32) and 2*phi (fp16).  Times a
torch.distributed NCCL allreduce of each size (CUDA events, max over ranks)
and reports algbw / busbw; the fused P2P exchange's own link bytes per rank
(4n(G-1)/G per direction) are listed beside it.

    python -m torch.distributed.run --nproc-per-node 4 tools/allreduce_sweep.py
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_05045_b200 import samo, workloads  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    G = dist.get_world_size()
    wl = workloads.gpt_2_7b()
    phi = wl.phi
    out = []
    for p in (0.5, 0.6, 0.7, 0.8, 0.9, 0.95, None):
        if p is None:
            cases = [("dense_fp32", 4 * phi, torch.float32), ("dense_fp16", 2 * phi, torch.float16)]
        else:
            n = sum(t.numel if not t.prunable else samo.unpruned_count(p, t.numel) for t in wl.tensors)
            cases = [(f"compressed_fp32_p{p}", 4 * n, torch.float32)]
        for name, nbytes, dt in cases:
            x = torch.ones(nbytes // torch.empty(0, dtype=dt).element_size(), dtype=dt, device="cuda")
            for _ in range(3):
                dist.all_reduce(x)
            torch.cuda.synchronize()
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 5
            a.record()
            for _ in range(reps):
                dist.all_reduce(x)
            b.record()
            torch.cuda.synchronize()
            t = torch.tensor([a.elapsed_time(b) / reps], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            row = {"G": G, "case": name, "bytes": nbytes, "ms": ms,
                   "algbw_GBps": nbytes / (ms * 1e-3) / 1e9,
                   "busbw_GBps": nbytes * 2 * (G - 1) / G / (ms * 1e-3) / 1e9}
            if p is not None:
                row["p2p_link_bytes_per_direction"] = (nbytes // 4) * 4 * (G - 1) // G
            out.append(row)
            del x
            torch.cuda.empty_cache()
    if dist.get_rank() == 0:
        for r in out:
            print(json.dumps(r))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
