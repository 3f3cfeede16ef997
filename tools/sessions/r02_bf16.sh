#!/bin/bash
# 1-GPU: parity (incl. bf16 gradients, local-group P2P, the C++ mirror KATs and
# the reference's store_test), bench lines for binary16 and bfloat16 grads.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out
T=${TAG:-r02f}
timeout 1500 python -m pytest tests -m gpu -q -rs -x > $O/${T}_pytest.log 2>&1; echo "rc=$?" >> $O/${T}_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/${T}_bench_n1.json 2> $O/${T}_bench_n1.err
timeout 600 python bench.py --steps 20 --warmup 5 --grad-dtype bf16 --no-cpu-baseline > $O/${T}_bench_bf16.json 2> $O/${T}_bench_bf16.err
echo done
