#!/bin/bash
# G = 2: P2P step with 1 bucket (serial, NCCL flag barrier; the default) vs
# the pipelined schedule with 4 / 8 buckets.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
: > gpurun_out/r02bk_g2.log
for B in 1 8 4 1 8 4; do
  SAMO_P2P_BUCKETS=$B timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700+B)) bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'B': $B, 'ms': d['ms_per_step'], 'pipe': d['pipeline_phases_ms'], 'overlap': (d['backward_overlap'] or {}).get('step_after_sinks_ms')}))" >> gpurun_out/r02bk_g2.log
done
echo done
