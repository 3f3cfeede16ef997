# Tuning sweep: tile size x CTAs/SM (1 GPU).  SWEEP="tile carve ctas" ...
mkdir -p gpurun_out
run() {
  echo "tile=$1 carve=$2 ctas=$3" >> gpurun_out/sweep.log
  SAMO_CARVEOUT=$2 SAMO_CTAS_PER_SM=$3 timeout 300 python bench.py --profile --steps 30 --warmup 3 --tile $1 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],4), {k: (round(v['ms'],4), round(v['frac'],3)) for k,v in d['kernels'].items()})" >> gpurun_out/sweep.log 2>&1
}
for cfg in ${SWEEP:-"8192 - 0" "4096 - 0" "16384 - 0" "8192 - 1"}; do
  set -- $cfg
  c=$2; [ "$c" = "-" ] && c=""
  run $1 "$c" $3
done
