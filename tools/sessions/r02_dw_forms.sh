#!/bin/bash
# dW GEMM forms per shape: auto, MS=1 (256x256 + tail split), MS=2 (512x256).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
: > gpurun_out/r02w_dw_forms.log
for F in auto 1 2 auto; do
  if [ "$F" = auto ]; then E=""; else E="SAMO_DW_MS=$F"; fi
  env $E timeout 300 python tools/bench_dw.py --reps 20 2>&1 | sed "s|^|ms=$F |" >> gpurun_out/r02w_dw_forms.log
done
echo done
