#!/bin/bash
# End-of-round check on a 4-GPU box: the multi-GPU tests the 2-GPU run
# skipped (G = 3, 4 across processes), the N = 4 and N = 1 bench lines.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dp.py -q -m gpu -rs -k "four_gpus or nccl_tolerance or three or across_devices" > gpurun_out/r02z_final_gpu4_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02z_final_gpu4_pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29543 \
  bench.py --gpus 4 > gpurun_out/r02z_final_bench_n4.json 2> gpurun_out/r02z_final_bench_n4.err
echo "bench4 rc=$?"
timeout 900 python bench.py > gpurun_out/r02z_final4_bench_n1.json 2> gpurun_out/r02z_final4_bench_n1.err
echo "bench1 rc=$?"
for f in gpurun_out/r02z_final_bench_n4.json gpurun_out/r02z_final4_bench_n1.json; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['ms_per_step'], d['value'], d.get('e2e',{}).get('value'), d.get('clocks'))"; done
