#!/bin/bash
# Final 4-GPU evidence: the whole -m gpu suite, then bench lines at N = 1, 2, 4
# and the reference arm.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out
T=${TAG:-r02q}
timeout 2400 python -m pytest tests -m gpu -q -rs > $O/${T}_gpu4_pytest.log 2>&1; echo "rc=$?" >> $O/${T}_gpu4_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/${T}_bench_n1.json 2> $O/${T}_bench_n1.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/${T}_ref_n1.json 2> $O/${T}_ref_n1.err
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500+N)) \
    bench.py --gpus $N --steps 20 --warmup 5 > $O/${T}_bench_n$N.json 2> $O/${T}_bench_n$N.err
done
echo done
