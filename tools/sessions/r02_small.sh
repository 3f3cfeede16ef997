#!/bin/bash
# 1-GPU: K123 short-step changes — parity, the checked suite subset, the bench
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out
T=${TAG:-r02r}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_state.py tests/test_cpp_kat.py -q -x > $O/${T}_pytest.log 2>&1; echo "rc=$?" >> $O/${T}_pytest.log
SAMO_LIB=$PWD/paper_2302_05045_b200/libsamo_cuda_checked.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $O/${T}_checked.log 2>&1; echo "rc=$?" >> $O/${T}_checked.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e > $O/${T}_bench_n1.json 2> $O/${T}_bench_n1.err
echo done
