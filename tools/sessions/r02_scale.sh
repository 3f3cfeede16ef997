#!/bin/bash
# 4-GPU: bench lines at N = 2 and 4 (binary16, default flags) and N = 4 bf16.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out
T=${TAG:-r02n}
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500+N)) \
    bench.py --gpus $N --steps 20 --warmup 5 > $O/${T}_bench_n$N.json 2> $O/${T}_bench_n$N.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 4 --steps 20 --warmup 5 --grad-dtype bf16 --no-e2e > $O/${T}_bench_n4_bf16.json 2> $O/${T}_bench_n4_bf16.err
echo done
