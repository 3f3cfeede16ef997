"""A/B of dW GEMM launch knobs (environment variables the launcher reads on
every call, e.g. SAMO_DW_MS, SAMO_DW_TAIL) in one process, interleaved over
rounds so clocks affect every variant alike; cuBLAS (x.T @ dy) alongside.
Each argument is one variant: space-separated NAME=VALUE assignments.

    python tools/ab_dw_env.py "SAMO_DW_MS=2" "SAMO_DW_MS=1" "SAMO_DW_MS=3 SAMO_DW_W_EW=1"
"""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2302_05045_b200 import samo  # noqa: E402
from tools.bench_dw import SHAPES, timed  # noqa: E402

EXTRA = [(4096, 2048, 2048), (4096, 2048, 8192), (4096, 8192, 2048), (2048, 4096, 4096)]


def main():
    variants = sys.argv[1:]
    keys = sorted({kv.split("=")[0] for v in variants for kv in v.split()})
    torch.manual_seed(0)
    for batch, n_in, n_out in SHAPES + EXTRA:
        x = (torch.rand(batch, n_in, device="cuda") * 2 - 1).half()
        dy = (torch.rand(batch, n_out, device="cuda") * 2 - 1).half()
        best = {v: float("inf") for v in variants + ["cublas"]}
        for _ in range(5):
            for v in variants:
                for k in keys:
                    os.environ.pop(k, None)
                for kv in v.split():
                    k, val = kv.split("=")
                    os.environ[k] = val
                best[v] = min(best[v], timed(lambda: samo.dw_gemm(x, dy), 20))
            best["cublas"] = min(best["cublas"], timed(lambda: torch.matmul(x.t(), dy), 20))
        fl = 2.0 * batch * n_in * n_out
        print(json.dumps({"shape": [batch, n_in, n_out],
                          "ms": {v: round(t, 4) for v, t in best.items()},
                          "of_cublas": {v: round(best["cublas"] / t, 3) for v, t in best.items() if v != "cublas"},
                          "tflops": {v: round(fl / t / 1e9, 1) for v, t in best.items()}}), flush=True)


if __name__ == "__main__":
    main()
