#!/bin/bash
# 4-GPU lease, second pass: the two tests fixed after r02h, bench lines at
# N = 2 and 4 (binary16 and bfloat16), and one attempt at NVLink link
# counters of the fused P2P kernels (rank 0 under ncu, G = 2, bounded).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out
T=${TAG:-r02k}
timeout 900 python -m pytest tests/test_gpu_dp.py -q -rs -k "sharded-bf16 or push_sinks or push_dw" > $O/${T}_gpu4_fixed.log 2>&1; echo "rc=$?" >> $O/${T}_gpu4_fixed.log
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500+N)) \
    bench.py --gpus $N --steps 20 --warmup 5 > $O/${T}_bench_n$N.json 2> $O/${T}_bench_n$N.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 4 --steps 20 --warmup 5 --grad-dtype bf16 --no-e2e > $O/${T}_bench_n4_bf16.json 2> $O/${T}_bench_n4_bf16.err
SAMO_SPIN_TIMEOUT_S=240 NCU_COUNT=3 timeout 480 python tools/launch_ncu_rank0.py 2 $O/${T}_nvlink_g2 -- \
  python bench.py --gpus 2 --steps 1 --warmup 3 --profile > $O/${T}_nvlink_g2.log 2>&1; echo "rc=$?" >> $O/${T}_nvlink_g2.log
ncu -i $O/${T}_nvlink_g2.ncu-rep --page raw --csv > $O/${T}_nvlink_g2_raw.csv 2>&1
echo done
