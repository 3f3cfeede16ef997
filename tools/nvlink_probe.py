#!/usr/bin/env python
"""Calibrates the NVML NVLink byte counters (paper_2302_05045_b200/nvlink.py)
against peer copies of known size: GPU 0 -> GPU 1, 1 GiB at a time, then the
counters of both GPUs are read.  One JSON line per repetition."""
from __future__ import annotations

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2302_05045_b200.nvlink import NvlinkBytes  # noqa: E402


def main() -> None:
    assert torch.cuda.device_count() >= 2
    c0, c1 = NvlinkBytes(0), NvlinkBytes(1)
    nbytes = 1 << 30
    a = torch.empty(nbytes, dtype=torch.uint8, device="cuda:0").fill_(1)
    b = torch.empty(nbytes, dtype=torch.uint8, device="cuda:1")
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    for rep in range(3):
        t0, r0 = c0.read(), c1.read()
        for _ in range(4):
            b.copy_(a)  # peer copy over NVLink (copy engine)
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        t1, r1 = c0.read(), c1.read()
        print(json.dumps({"rep": rep, "source": c0.source, "links": len(c0.links), "copied": 4 * nbytes,
                          "gpu0_tx": t1[0] - t0[0], "gpu0_rx": t1[1] - t0[1],
                          "gpu1_tx": r1[0] - r0[0], "gpu1_rx": r1[1] - r0[1]}))


if __name__ == "__main__":
    main()
