#!/bin/bash
# 1-GPU: the speculative P2P step in one-GPU local groups (incl. skip repair,
# sinks, bf16) + the non-spec local-group suite as a regression check.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_dp.py -q -x -k "local_group" > $O/r02o_spec_local.log 2>&1; echo "rc=$?" >> $O/r02o_spec_local.log
echo done
