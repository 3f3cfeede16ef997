#!/bin/bash
# K123 v2 (dynamic tiles, deferred copy-out): parity + bench at two tile sizes.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out
T=${TAG:-r02c}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_state.py -x -q > $O/${T}_pytest.log 2>&1; echo "rc=$?" >> $O/${T}_pytest.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/${T}_bench_t16k.json 2> $O/${T}_bench_t16k.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --tile 8192 > $O/${T}_bench_t8k.json 2> $O/${T}_bench_t8k.err
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > $O/${T}_fullsize.log 2>&1; echo "rc=$?" >> $O/${T}_fullsize.log
echo done
