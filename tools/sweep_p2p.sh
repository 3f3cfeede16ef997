# k_shard_p2p occupancy variants (libsamo_cuda_p2p{2,3,4}.so built with
# -DSAMO_P2P_MINB/GRID) vs the default build, at NGPU GPUs.
mkdir -p gpurun_out
N=${NGPU:-2}
for lib in libsamo_cuda.so libsamo_cuda_p2p2.so libsamo_cuda_p2p3.so libsamo_cuda_p2p4.so; do
  echo "G=$N lib=$lib" >> gpurun_out/sweep_p2p.log
  SAMO_LIB=$PWD/paper_2302_05045_b200/$lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 2000)) bench.py --gpus $N --steps 30 --warmup 3 --no-e2e 2>/dev/null \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d.get('phases_ms'))" >> gpurun_out/sweep_p2p.log 2>&1
done
