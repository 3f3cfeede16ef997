# BASELINE.json configs 1-3 on one GPU: FC sweep (incl. config 1 = fc4096) and
# the GPT-1.3B set at three sparsities.  One JSON line per run in
# gpurun_out/r02_configs.jsonl.
mkdir -p gpurun_out
for n in 128 256 512 1024 2048 4096; do
  timeout 300 python bench.py --workload fc$n --steps 500 --warmup 20 --no-e2e --no-cpu-baseline --no-fused --graph 2>/dev/null | tail -1 >> gpurun_out/r02_configs.jsonl
done
for p in 0.8 0.9 0.95; do
  timeout 300 python bench.py --workload gpt-1.3b --sparsity $p --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-fused 2>/dev/null | tail -1 >> gpurun_out/r02_configs.jsonl
done
for p in 0.5 0.8 0.95; do
  timeout 300 python bench.py --workload gpt-2.7b --sparsity $p --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-fused 2>/dev/null | tail -1 >> gpurun_out/r02_configs.jsonl
done
