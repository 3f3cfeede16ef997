#!/bin/bash
# The data-parallel suite on a 4-GPU box after removing the losing P2P variants.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dp.py -q -m gpu -x -rs > gpurun_out/r02z_dp4_pytest.log 2>&1
echo "pytest rc=$?"
tail -3 gpurun_out/r02z_dp4_pytest.log
