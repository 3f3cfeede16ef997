#!/bin/bash
# 4-GPU lease (gpurun --gpus 4): the whole -m gpu suite (every cross-process
# DP test runs), bench lines N = 1, 2, 4 and the reference arm, NVLink link
# counters of the fused P2P kernels (rank 0 under ncu, G = 2 and 4), NVLink
# tools probe.  Outputs under gpurun_out/ (copied to profiles/).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out
T=${TAG:-r02h}
nvidia-smi topo -m > $O/${T}_topo.txt 2>&1
(nvidia-smi nvlink -s -i 0; nvidia-smi nvlink -gt d -i 0) > $O/${T}_nvsmi_nvlink.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs > $O/${T}_gpu4_pytest.log 2>&1; echo "rc=$?" >> $O/${T}_gpu4_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/${T}_bench_n1.json 2> $O/${T}_bench_n1.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/${T}_ref_n1.json 2> $O/${T}_ref_n1.err
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500+N)) \
    bench.py --gpus $N --steps 20 --warmup 5 > $O/${T}_bench_n$N.json 2> $O/${T}_bench_n$N.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 4 --steps 20 --warmup 5 --grad-dtype bf16 --no-e2e > $O/${T}_bench_n4_bf16.json 2> $O/${T}_bench_n4_bf16.err
for G in 2 4; do
  SAMO_SPIN_TIMEOUT_S=1200 NCU_COUNT=4 timeout 1500 python tools/launch_ncu_rank0.py $G $O/${T}_nvlink_g$G -- \
    python bench.py --gpus $G --steps 2 --warmup 3 --profile > $O/${T}_nvlink_g$G.log 2>&1; echo "rc=$?" >> $O/${T}_nvlink_g$G.log
  ncu -i $O/${T}_nvlink_g$G.ncu-rep --page raw --csv > $O/${T}_nvlink_g${G}_raw.csv 2>&1
done
echo done
