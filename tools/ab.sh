# A/B: an older build vs the current tree, alternating on the same box.
# Prepare: git worktree add ab_old <commit> && (cd ab_old && python -m paper_2302_05045_b200.build)
mkdir -p gpurun_out
for i in 1 2; do
  for d in ab_old .; do
    (cd $d && timeout 300 python bench.py --profile --steps 40 --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d', round(d['ms_per_step'],4), {k: round(v['ms'],4) for k,v in d['kernels'].items()})") >> gpurun_out/ab.log 2>&1
  done
done
