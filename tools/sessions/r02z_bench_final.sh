#!/bin/bash
# Final bench lines (N = 1 and N = 2) with the NVML clock sampler.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
[ -n "$SKIP1" ] || timeout 900 python bench.py > gpurun_out/r02z_bench_final_n1.json 2> gpurun_out/r02z_bench_final_n1.err
echo "bench1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 \
  bench.py --gpus 2 > gpurun_out/r02z_bench_final_n2.json 2> gpurun_out/r02z_bench_final_n2.err
echo "bench2 rc=$?"
for f in gpurun_out/r02z_bench_final_n1.json gpurun_out/r02z_bench_final_n2.json; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['ms_per_step'], d['unsampled'], d['value'], d.get('e2e',{}).get('value'), d.get('clocks'), d.get('roofline',{}).get('frac'))"; done
