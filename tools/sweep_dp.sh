# DP overlap sweep on the GPUs of this call: reserve SMs x NCCL CTA cap x buckets.
mkdir -p gpurun_out
N=${NGPU:-2}
for cfg in ${DPSWEEP:-"16 0 8" "24 0 8" "32 0 8" "16 16 8" "24 24 8" "16 0 4" "0 0 1"}; do
  set -- $cfg
  echo "reserve=$1 maxctas=$2 buckets=$3 overlap=$([ $3 = 1 ] && echo 0 || echo 1)" >> gpurun_out/sweep_dp.log
  extra=""
  [ "$2" != "0" ] && extra="NCCL_MAX_CTAS=$2"
  env SAMO_NCCL_SMS=$1 SAMO_BUCKETS=$3 SAMO_OVERLAP=$([ $3 = 1 ] && echo 0 || echo 1) $extra timeout 300 \
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
    bench.py --gpus $N --steps 30 --warmup 3 --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k: round(v['ms'],4) for k,v in d['kernels'].items()})" >> gpurun_out/sweep_dp.log 2>&1
done
