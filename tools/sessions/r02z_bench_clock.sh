#!/bin/bash
# N = 1 bench: 50 steps (the default) and 20, after the clock sampler waits for
# its first sample before the timed region starts.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for st in 50 20 50; do
  timeout 600 python bench.py --steps $st --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print($st, d['ms_per_step'], d['kernels']['K123_fused_step']['ms'], d['clocks'])" >> gpurun_out/r02z_bench_clock.log
done
cat gpurun_out/r02z_bench_clock.log
