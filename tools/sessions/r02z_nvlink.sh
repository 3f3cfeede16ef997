#!/bin/bash
# NVLink bytes of the fused P2P kernels: a multi-device local group (one
# process, one model per GPU) under ncu with the link counters.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
G=${G:-2}
nvidia-smi topo -m > gpurun_out/r02z_topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_dp.py -q -m gpu -k "local_group" -x > gpurun_out/r02z_pytest_g$G.log 2>&1
echo "pytest rc=$?"
timeout 300 python tools/nvlink_group_ncu.py $G > gpurun_out/r02z_plain_g$G.log 2>&1
echo "plain rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  -k regex:"k1_gather|k_shard_p2p" --clock-control none --csv \
  --log-file gpurun_out/r02z_nvlink_g$G.csv python tools/nvlink_group_ncu.py $G > gpurun_out/r02z_ncu_g$G.log 2>&1
echo "ncu rc=$?"
