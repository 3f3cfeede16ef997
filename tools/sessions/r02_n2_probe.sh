#!/bin/bash
# 2-GPU: the data-parallel bench with and without the NVML NVLink reads, and
# with the phase-timed pass only, to find the N > 1 regression.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out
: > $O/r02m_n2.log
for V in 0 1 0; do
  SAMO_BENCH_NVLINK=$V timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29600+V)) bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e 2> $O/r02m_n2_$V.err | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'nvml': $V, 'ms': d['ms_per_step'], 'phases': d['phases_ms'], 'overlap': d['backward_overlap']}))" >> $O/r02m_n2.log
done
nvidia-smi -q -d PERFORMANCE,CLOCK | head -60 > $O/r02m_smi.txt
echo done
