#!/bin/bash
# dW GEMM after the 256 x 384 form joined the automatic choice: parity, the
# auto choice against each form, and the bench_dw table.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dw.py -q -m gpu -x > gpurun_out/r02z_dw2_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/r02z_dw2_pytest.log
timeout 900 python tools/ab_dw_env.py "" "SAMO_DW_MS=2" "SAMO_DW_MS=1" "SAMO_DW_MS=3" > gpurun_out/r02z_dw2_ab.jsonl 2>&1
echo "ab rc=$?"
timeout 900 python tools/bench_dw.py > gpurun_out/r02z_bench_dw.jsonl 2>&1
echo "bench_dw rc=$?"; cat gpurun_out/r02z_bench_dw.jsonl
