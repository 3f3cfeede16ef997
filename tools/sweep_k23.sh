# K23 variant sweep (chunk, stages) at T=8192 and 16384 + the HBM mix probe.
mkdir -p gpurun_out
./tools/bw_probe 2 > gpurun_out/bw_probe.json 2>&1
for v in 0 1 2 3 4; do
  for t in 8192 16384; do
    echo "variant=$v tile=$t" >> gpurun_out/sweep.log
    SAMO_K23_VARIANT=$v timeout 300 python bench.py --profile --steps 30 --warmup 3 --tile $t 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],4), {k: (round(v['ms'],4), round(v['frac'],3)) for k,v in d['kernels'].items()})" >> gpurun_out/sweep.log 2>&1
  done
done
