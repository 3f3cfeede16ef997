# P2P step variants at NGPU GPUs: each VARIANT is a list of env assignments
# (SAMO_P2P_BUCKETS, SAMO_P2P_PUSH, SAMO_P2P_SHARD_CTAS, SAMO_P2P_EXPAND_CTAS).
mkdir -p gpurun_out
N=${NGPU:-4}
OUT=gpurun_out/sweep_p2p_pipe_g$N.log
IFS=';' read -ra VS <<< "${VARIANTS:-SAMO_P2P_BUCKETS=1 SAMO_P2P_PUSH=1;SAMO_P2P_BUCKETS=1 SAMO_P2P_PUSH=0;SAMO_P2P_BUCKETS=8 SAMO_P2P_PUSH=1;SAMO_P2P_BUCKETS=8 SAMO_P2P_PUSH=0}"
for v in "${VS[@]}"; do
  echo "$v" >> $OUT
  env $v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 2000)) bench.py --gpus $N --steps 30 --warmup 3 \
    --no-e2e --no-cpu-baseline ${EXTRA:-} 2>>gpurun_out/sweep_p2p_pipe.err \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d.get('p2p_features'), d.get('pipeline_phases_ms'), d.get('phases_ms'))" >> $OUT 2>&1
done
