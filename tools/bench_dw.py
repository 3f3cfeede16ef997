"""Weight-gradient GEMM + backward sink timings (1 GPU), one JSON line per shape.

    python tools/bench_dw.py [--p 0.9] [--reps 20]

For each (batch, in, out): our tcgen05 dW GEMM (dense binary16 out), cuBLAS
via torch.matmul(x.T, dy) for reference, the unfused sink (dense dW GEMM ->
K1 on the layer) and the fused sink (GEMM with the gather in its epilogue).
CUDA events around --reps back-to-back calls (best of 3), inputs resident in HBM.
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2302_05045_b200 import samo  # noqa: E402

SHAPES = [  # (batch tokens, in, out)
    (576, 4096, 4096),      # config 2's largest FC layer at batch 576
    (4096, 2560, 10240),    # GPT-2.7B MLP up
    (4096, 10240, 2560),    # GPT-2.7B MLP down
    (4096, 2560, 7680),     # GPT-2.7B attention qkv
    (4096, 2560, 2560),     # GPT-2.7B attention out
    (8192, 2560, 10240),
]


def timed(fn, reps):
    """Device time per call: `reps` calls queued back to back between two
    events (host launch overhead overlaps the previous call), best of 3."""
    for _ in range(3):
        fn()
    best = float("inf")
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) / reps)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=float, default=0.9)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    torch.manual_seed(0)
    for batch, n_in, n_out in SHAPES:
        x = (torch.rand(batch, n_in, device="cuda") * 2 - 1).half()
        dy = ((torch.rand(batch, n_out, device="cuda") * 2 - 1) * 4).half()
        n = n_in * n_out
        keep = int(round((1 - args.p) * n))
        idx = torch.randperm(n, device="cuda")[:keep].sort().values.to(torch.int32)
        m = samo.SamoModel.from_index_sets([samo.PrunedIndexSet("fc.weight", n, idx)], [(n_in, n_out)], 0)
        m.init_layer(0, torch.zeros(n, device="cuda"))
        flops = 2.0 * batch * n_in * n_out
        dense = samo.dw_gemm(x, dy).reshape(-1)
        t_k1 = timed(lambda: m.sink_dense(0, dense), args.reps)
        # the four contenders round-robin (best of 5 rounds each), so that
        # power-capped clocks under sustained tensor load hit all alike
        fns = {"gemm": lambda: samo.dw_gemm(x, dy), "cublas": lambda: torch.matmul(x.t(), dy),
               "unfused": lambda: m.sink_dense(0, samo.dw_gemm(x, dy).reshape(-1)),
               "fused": lambda: m.sink_dw(0, x, dy)}
        best = {k: float("inf") for k in fns}
        for _ in range(5):
            for k, fn in fns.items():
                best[k] = min(best[k], timed(fn, args.reps))
            m._sink_keepalive.clear()
        t_ours, t_cublas, t_unfused, t_fused = best["gemm"], best["cublas"], best["unfused"], best["fused"]
        print(json.dumps({
            "batch": batch, "in": n_in, "out": n_out, "p": args.p,
            "dw_gemm_ms": round(t_ours, 4), "dw_gemm_tflops": round(flops / t_ours / 1e9, 1),
            "cublas_ms": round(t_cublas, 4), "cublas_tflops": round(flops / t_cublas / 1e9, 1),
            "k1_layer_ms": round(t_k1, 4),
            "unfused_sink_ms": round(t_unfused, 4), "fused_sink_ms": round(t_fused, 4),
            "fused_saving": round(1 - t_fused / t_unfused, 3),
        }), flush=True)
        del m


if __name__ == "__main__":
    main()
