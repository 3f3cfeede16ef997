# Tuning sweep over tile size (1 GPU): TILES="8192 16384" bash tools/sweep_tiles.sh
mkdir -p gpurun_out
for t in ${TILES:-8192 16384 4096}; do
  echo "tile=$t ctas=${SAMO_CTAS_PER_SM:-auto}" >> gpurun_out/sweep.log
  timeout 300 python bench.py --profile --steps 30 --warmup 3 --tile $t 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],4), {k: (round(v['ms'],4), round(v['frac'],3)) for k,v in d['kernels'].items()})" >> gpurun_out/sweep.log 2>&1
done
