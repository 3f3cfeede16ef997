#!/bin/bash
# N = 4 bench over 20 and 50 timed steps, alternated (run-length effect).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for st in 20 50 20 50 100; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + st)) \
    bench.py --gpus 4 --steps $st --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print($st, round(d['ms_per_step'],4), d.get('pipeline_phases_ms'), d['clocks'])" >> gpurun_out/r02z_n4_steps.log
done
cat gpurun_out/r02z_n4_steps.log
