#!/usr/bin/env python
"""Runs a data-parallel command on G local GPUs (one process per GPU, the env
torch.distributed.run would set) with rank 0 alone under ncu, so the fused
NVLink kernels can be profiled in a real cross-process group.

    python tools/launch_ncu_rank0.py G NCU_OUT_BASE -- python bench.py --gpus G ...

ncu on rank 0 uses kernel replay with a short metric list (duration, DRAM and
NVLink tx/rx user bytes) filtered to the K1 push and shard kernels, so each
profiled launch replays a handful of times.  Replays are safe here: K1's
peer stores and the shard kernel's peer stores / bucket signals are
idempotent (same values, same epochs), and ncu restores rank 0's own memory
between passes.  The other ranks wait in their peer-signal spins meanwhile
(30 s trap, far above the capture time).  Numbers printed by the profiled
run are not bench values."""
from __future__ import annotations

import os
import socket
import subprocess
import sys

METRICS = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
           "nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum")


def main() -> None:
    G = int(sys.argv[1])
    out = sys.argv[2]
    cmd = sys.argv[sys.argv.index("--") + 1:]
    kfilter = os.environ.get("NCU_KERNELS", "regex:k1_gather|k_shard_p2p")
    count = os.environ.get("NCU_COUNT", "6")
    plain_first = os.environ.get("NCU_PLAIN_FIRST", "1") != "0"
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = []
    for r in range(G):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(G), LOCAL_WORLD_SIZE=str(G),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        c = list(cmd)
        if r == 0:
            c = ["ncu", "--metrics", METRICS, "--clock-control", "none", "-k", kfilter, "-c", count,
                 "-f", "-o", out] + c
        elif plain_first:
            # the pool's ncu first runs rank 0's command once without ncu: the
            # other ranks take part in that run and then in the profiled one
            c = ["bash", "-c", " ".join(cmd) + " && " + " ".join(cmd)]
        procs.append(subprocess.Popen(c, env=env))
    rc = 0
    for p in procs:
        rc = p.wait() or rc
    sys.exit(rc)


if __name__ == "__main__":
    main()
