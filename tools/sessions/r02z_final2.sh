#!/bin/bash
# End-of-round check on a 2-GPU box: the whole -m gpu suite, then the N = 1
# and N = 2 bench lines.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rs > gpurun_out/r02z_final_gpu2_pytest.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/r02z_final_gpu2_pytest.log
timeout 900 python bench.py > gpurun_out/r02z_final_bench_n1.json 2> gpurun_out/r02z_final_bench_n1.err
echo "bench1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 \
  bench.py --gpus 2 > gpurun_out/r02z_final_bench_n2.json 2> gpurun_out/r02z_final_bench_n2.err
echo "bench2 rc=$?"
for f in gpurun_out/r02z_final_bench_n1.json gpurun_out/r02z_final_bench_n2.json; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['ms_per_step'], d['value'], d.get('e2e',{}).get('value'), d.get('roofline',{}).get('frac'))"; done
