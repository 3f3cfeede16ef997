#!/bin/bash
# A/B: K123 skipping all-pruned theta16 sectors (current tree) vs HEAD (ab_s),
# plus the parity tests of the current tree.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r02s_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02s_pytest.log
BENCH_ARGS="--sparsity 0.9" bash tools/ab3.sh ab_s . > /dev/null 2>&1; cp gpurun_out/ab3.log gpurun_out/r02s_ab_p09.log
BENCH_ARGS="--sparsity 0.95" bash tools/ab3.sh ab_s . > /dev/null 2>&1; cp gpurun_out/ab3.log gpurun_out/r02s_ab_p095.log
echo done
