#!/bin/bash
# The 256 x 384 dW pair tile: parity of every form, then an interleaved A/B.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dw.py -q -m gpu -x > gpurun_out/r02z_dw_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02z_dw_pytest.log
timeout 900 python tools/ab_dw_env.py "" "SAMO_DW_MS=2" "SAMO_DW_MS=1" "SAMO_DW_MS=3" "SAMO_DW_MS=3 SAMO_DW_W_EW=1" > gpurun_out/r02z_dw_ab.jsonl 2>&1
echo "ab rc=$?"; cat gpurun_out/r02z_dw_ab.jsonl
