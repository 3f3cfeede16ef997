# Data-parallel bench on NGPU GPUs for each exchange mode in MODES.
mkdir -p gpurun_out
N=${NGPU:-2}
for m in ${MODES:-sharded allreduce}; do
  SAMO_EXCHANGE=$m timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 2000)) \
    bench.py --gpus $N --steps ${STEPS:-30} --warmup 3 ${EXTRA:---no-e2e} > gpurun_out/bench${N}_$m.log 2>&1
  echo "$m rc=$?" >> gpurun_out/bench_dp.log
done
