# Sharded DP sweep: reserve SMs x buckets at NGPU GPUs.
mkdir -p gpurun_out
N=${NGPU:-4}
for cfg in ${SHSWEEP:-"0:4" "16:4" "24:4" "32:4" "24:8" "24:2" "32:8"}; do
  R=${cfg%%:*}; B=${cfg##*:}
  echo "G=$N reserve=$R buckets=$B" >> gpurun_out/sweep_shard.log
  SAMO_SHARD_NCCL_SMS=$R SAMO_SHARD_BUCKETS=$B timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 2000)) bench.py --gpus $N --steps 30 --warmup 3 --no-e2e 2>/dev/null \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d.get('phases_ms'))" >> gpurun_out/sweep_shard.log 2>&1
done
