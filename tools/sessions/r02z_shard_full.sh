#!/bin/bash
# Full ncu capture of K1 (push) and k_shard_p2p in the two-GPU one-process
# group (third step; SAMO_P2P_BUCKETS=2: per step K1 r0, K1 r1, then two
# shard launches per rank).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
export SAMO_P2P_BUCKETS=2
timeout 300 python tools/nvlink_group_ncu.py 2 > gpurun_out/r02z_full_plain.log 2>&1
echo "plain rc=$?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k1_gather|k_shard_p2p" \
  --launch-skip 12 -c 3 -o gpurun_out/r02z_k1_shard_g2 -f python tools/nvlink_group_ncu.py 2 > gpurun_out/r02z_full_ncu.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/r02z_full_ncu.log
