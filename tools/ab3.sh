#!/bin/bash
# A/B/C: worktrees given as arguments (each built in place), alternating on
# the same box; one summary line per run into gpurun_out/ab3.log.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/ab3.log
for i in 1 2; do
  for d in "$@"; do
    (cd $d && timeout 300 python bench.py --profile --steps 40 --warmup 5 $BENCH_ARGS 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d', round(d['ms_per_step'],4), {k: round(v['ms'],4) for k,v in d['kernels'].items()})") >> gpurun_out/ab3.log 2>&1
  done
done
cat gpurun_out/ab3.log
