#!/bin/bash
# dW GEMM stream-K tail: correctness, then timings with SAMO_DW_SK=0/1.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_dw.py tests/test_cpp_kat.py -q -x > $O/r02sk_pytest.log 2>&1; echo "rc=$?" >> $O/r02sk_pytest.log
: > $O/r02sk_dw.log
for V in 0 1 0 1; do
  SAMO_DW_SK=$V timeout 300 python tools/bench_dw.py --reps 20 2>&1 | sed "s|^|sk=$V |" >> $O/r02sk_dw.log
done
echo done
