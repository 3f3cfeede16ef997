#!/bin/bash
# 256 x 384 form with three epilogue groups (one 128-column half each).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dw.py -q -m gpu -x > gpurun_out/r02z_dw_ew3_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/r02z_dw_ew3_pytest.log
timeout 600 python tools/ab_dw_env.py "SAMO_DW_MS=3" "SAMO_DW_MS=3 SAMO_DW_W_EW=3" "SAMO_DW_MS=2" > gpurun_out/r02z_dw_ew3_ab.jsonl 2>&1
echo "ab rc=$?"
python -c "
import json
for l in open('gpurun_out/r02z_dw_ew3_ab.jsonl'):
    d=json.loads(l); print(d['shape'], d['of_cublas'])"
