#!/bin/bash
# Round-2 multi-GPU evidence on a 4-GPU lease (gpurun --gpus 4): NCCL
# tolerance tests, NVLink counter calibration, bench lines at N = 1, 2, 4 and
# the reference arm, ncu NVLink bytes of the fused kernels at G = 4, and the
# config-5 allreduce sweep.  Outputs under gpurun_out/ (copied to profiles/).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_dp.py -q -rs -k "nccl or refused" > $O/r02_dp_nccl.log 2>&1; echo "rc=$?" >> $O/r02_dp_nccl.log
timeout 300 python tools/nvlink_probe.py > $O/r02_nvlink_probe.jsonl 2> $O/r02_nvlink_probe.err
timeout 600 python bench.py --steps 20 --warmup 5 > $O/r02_bench_n1.json 2> $O/r02_bench_n1.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/r02_ref_n1.json 2> $O/r02_ref_n1.err
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500+N)) \
    bench.py --gpus $N --steps 20 --warmup 5 > $O/r02_bench_n$N.json 2> $O/r02_bench_n$N.err
done
timeout 600 python tools/launch_ncu_rank0.py 4 $O/r02_nvlink_g4 -- python bench.py --gpus 4 --steps 2 --warmup 3 --profile > $O/r02_nvlink_g4.log 2>&1; echo "rc=$?" >> $O/r02_nvlink_g4.log
ncu -i $O/r02_nvlink_g4.ncu-rep --page raw --csv > $O/r02_nvlink_g4_raw.csv 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29600 \
  tools/allreduce_sweep.py > $O/r02_ar_sweep_g4.jsonl 2> $O/r02_ar_sweep_g4.err
echo done
