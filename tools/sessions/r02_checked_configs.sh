#!/bin/bash
# 1-GPU: the -m gpu suite against the CHECKED library (device bounds checks,
# trapping waits; compute-sanitizer is closed on this pool), then the
# BASELINE config-3 bench lines (GPT-1.3B at p = 0.8 / 0.9 / 0.95) and the
# GPT-2.7B sparsity variants.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out
T=${TAG:-r02i}
SAMO_LIB=$PWD/paper_2302_05045_b200/libsamo_cuda_checked.so timeout 2400 python -m pytest tests -m gpu -q -rs \
  > $O/${T}_checked_pytest.log 2>&1; echo "rc=$?" >> $O/${T}_checked_pytest.log
: > $O/${T}_configs.jsonl
for W in "gpt-1.3b 0.8" "gpt-1.3b 0.9" "gpt-1.3b 0.95" "gpt-2.7b 0.5" "gpt-2.7b 0.8" "gpt-2.7b 0.95"; do
  set -- $W
  timeout 600 python bench.py --workload $1 --sparsity $2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
    2>> $O/${T}_configs.err | tail -1 >> $O/${T}_configs.jsonl
done
echo done
