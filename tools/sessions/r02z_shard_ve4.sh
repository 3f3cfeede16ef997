#!/bin/bash
# Two-GPU check of the VE = 4 serial shard kernel: DP parity + the N = 2 bench line.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dp.py -q -m gpu -x -k "two_gpus or across_devices or local_group" > gpurun_out/r02z_ve4_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/r02z_ve4_pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 > gpurun_out/r02z_bench_n2.json 2> gpurun_out/r02z_bench_n2.err
echo "bench rc=$?"; tail -c 600 gpurun_out/r02z_bench_n2.json
