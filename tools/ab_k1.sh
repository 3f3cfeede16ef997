# A/B of an older build (git worktree at ab_old, built in place) vs the current tree at several sparsities (1 GPU).
mkdir -p gpurun_out
for p in ${PS:-0.9 0.5 0.8}; do
  for d in ab_old .; do
    (cd $d && timeout 300 python bench.py --profile --steps 30 --warmup 3 --sparsity $p 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d p=$p', round(d['ms_per_step'],4), {k: (round(v['ms'],4), round(v['frac'],3)) for k,v in d['kernels'].items()})") >> gpurun_out/ab.log 2>&1
  done
done
