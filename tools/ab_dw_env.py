"""A/B of a dW GEMM launch knob (an environment variable the launcher reads
on every call, e.g. SAMO_DW_MS, SAMO_DW_TAIL) in one process, interleaved
over rounds so clocks affect both alike.

    python tools/ab_dw_env.py SAMO_DW_MS 2 1
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
    var, a, b = sys.argv[1], sys.argv[2], sys.argv[3]
    torch.manual_seed(0)
    for batch, n_in, n_out in SHAPES + EXTRA:
        x = (torch.rand(batch, n_in, device="cuda") * 2 - 1).half()
        dy = (torch.rand(batch, n_out, device="cuda") * 2 - 1).half()
        best = {a: float("inf"), b: float("inf")}
        for _ in range(5):
            for t in (a, b):
                os.environ[var] = t
                best[t] = min(best[t], timed(lambda: samo.dw_gemm(x, dy), 20))
        fl = 2.0 * batch * n_in * n_out
        tiles = ((n_in + 255) // 256) * ((n_out + 255) // 256)
        print(json.dumps({"shape": [batch, n_in, n_out], "tiles256": tiles, var: [a, b],
                          "ms": [round(best[a], 4), round(best[b], 4)],
                          "tflops": [round(fl / best[a] / 1e9, 1), round(fl / best[b] / 1e9, 1)],
                          "t_b_over_t_a_minus_1": round(best[b] / best[a] - 1, 3)}), flush=True)


if __name__ == "__main__":
    main()
