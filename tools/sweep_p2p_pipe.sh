# Pipelined P2P step: buckets x grid split, at NGPU GPUs (one line per variant).
mkdir -p gpurun_out
N=${NGPU:-4}
OUT=gpurun_out/sweep_p2p_pipe_g$N.log
for v in ${VARIANTS:-"1 4 1" "4 4 1" "8 4 1" "4 2 1" "4 8 1" "4 4 2" "4 2 2" "8 2 2"}; do
  set -- $v
  echo "B=$1 shard_ctas=$2 expand_ctas=$3" >> $OUT
  SAMO_P2P_BUCKETS=$1 SAMO_P2P_SHARD_CTAS=$2 SAMO_P2P_EXPAND_CTAS=$3 timeout 300 \
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 2000)) bench.py --gpus $N --steps 30 --warmup 3 \
    --no-e2e --no-cpu-baseline ${EXTRA:-} 2>>gpurun_out/sweep_p2p_pipe.err \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d.get('pipeline_phases_ms'))" >> $OUT 2>&1
done
