#!/bin/bash
# 1-GPU check of the fused K123 step: the -m gpu suite, the bench line, the
# ncu launch list of the bench, and one ncu --set full capture of K123.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out
T=${TAG:-r02b}
timeout 1200 python -m pytest tests -m gpu -x -q > $O/${T}_pytest.log 2>&1; echo "rc=$?" >> $O/${T}_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/${T}_bench_n1.json 2> $O/${T}_bench_n1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${T}_launches.csv \
  python bench.py --steps 2 --warmup 3 --profile > $O/${T}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k123 -c 1 -o $O/${T}_k123 -f \
  python bench.py --steps 2 --warmup 3 --profile > $O/${T}_ncu_full.log 2>&1
echo done
