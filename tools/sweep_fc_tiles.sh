# Tile size vs small workloads (1 GPU, graph step): one line per (workload, tile).
mkdir -p gpurun_out
for w in ${WORKLOADS:-fc1024 fc2048 fc4096 gpt-1.3b}; do
  for t in ${TILES:-1024 2048 4096 8192 16384}; do
    s=500; [ "${w#gpt}" != "$w" ] && s=30
    r=$(timeout 300 python bench.py --workload $w --tile $t --steps $s --warmup 10 --no-e2e --no-cpu-baseline --graph 2>/dev/null | tail -1 \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,2), 'us', {k: round(v['ms']*1000,2) for k,v in d['kernels'].items()})")
    echo "$w tile=$t $r" >> gpurun_out/sweep_fc_tiles.log
  done
done
