#!/bin/bash
# 1-GPU: HBM ceilings (incl. the TMA bulk copy), the headline bench line,
# its ncu launch list and one ncu --set full capture of K123.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out
T=${TAG:-r02l}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bw_probe tools/bw_probe.cu && timeout 300 tools/bw_probe 2 > $O/${T}_bw_probe.jsonl 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $O/${T}_bench_n1.json 2> $O/${T}_bench_n1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${T}_launches.csv \
  python bench.py --steps 2 --warmup 3 --profile > $O/${T}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k123_step -c 1 -o $O/${T}_k123 -f \
  python bench.py --steps 2 --warmup 3 --profile > $O/${T}_ncu_full.log 2>&1
echo done
