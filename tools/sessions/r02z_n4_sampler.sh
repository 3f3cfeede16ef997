#!/bin/bash
# N = 4: the clock sampler's own effect on the step (SAMO_BENCH_CLOCKS modes).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
OUT=gpurun_out/${OUT:-r02z_n4_sampler.log}
for rep in ${REPS:-1 2}; do
  for mode in ${MODES:-off nvml nvml_power}; do
    SAMO_BENCH_CLOCKS=$mode timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NGPU:-4} \
      --master-addr 127.0.0.1 --master-port $((29700 + rep * 10 + RANDOM % 9)) bench.py --gpus ${NGPU:-4} --steps 50 --no-e2e \
      2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('clocks=$mode', round(d['ms_per_step'],4), d.get('clocks'))" >> $OUT
  done
done
cat $OUT
