#!/bin/bash
# A/B of k_shard_p2p builds (ab_shard/lib_*.so) at NGPU ranks:
# ms/step and the serial phase breakdown per run, alternating libraries.
# A variant library: compile csrc/kernels_fused.cu with the build.py flags
# plus its -D settings, then link it with the other in-tree objects, e.g.
#   nvcc <build.py NVCC_FLAGS> -DX=1 -I include -I csrc -c csrc/kernels_fused.cu -o /tmp/kf_X.o
#   nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab_shard/lib_X.so \
#        $(ls build/*.o | grep -v kernels_fused) /tmp/kf_X.o -lnccl -cudart static
# VARIANTS="A B:SAMO_P2P_SHARD_CTAS=4" runs lib_A, then lib_B with that env.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=${NGPU:-2}
OUT=gpurun_out/ab_shard_g$N.log
: > $OUT
for rep in 1 2; do
  for v in ${VARIANTS:-A B C}; do
    lib=${v%%:*}; env=""; [[ "$v" == *:* ]] && env=${v#*:}
    env SAMO_LIB=ab_shard/lib_$lib.so $env timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $N --steps 30 --warmup 5 \
      --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$v', round(d['ms_per_step'],4), d.get('phases_ms'), d.get('pipeline_phases_ms'))" >> $OUT 2>&1
  done
done
cat $OUT
