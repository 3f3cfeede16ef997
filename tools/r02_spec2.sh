#!/bin/bash
# N-GPU: cross-process tests of the speculative step, then bench A/B:
# default step vs SAMO_P2P_SPEC=1 with K1 at 1/2/3 CTAs per SM.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out
N=${N:-2}
T=${TAG:-r02p}
timeout 900 python -m pytest tests/test_gpu_dp.py -q -x -rs -k "spec and not local" > $O/${T}_spec_dp.log 2>&1; echo "rc=$?" >> $O/${T}_spec_dp.log
: > $O/${T}_spec_bench.jsonl
for V in "0 2" "1 1" "1 2" "1 3" "0 2"; do
  set -- $V
  SAMO_P2P_SPEC=$1 SAMO_P2P_SPEC_K1_CTAS=$2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29600 + $1 * 10 + $2)) bench.py --gpus $N --steps 20 --warmup 5 --no-e2e \
    2>> $O/${T}_spec_bench.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'spec': $1, 'k1_ctas': $2, 'ms': d['ms_per_step'], 'pipe': d['pipeline_phases_ms'], 'phases': d['phases_ms'], 'overlap': {k: v for k, v in (d['backward_overlap'] or {}).items() if k != 'note'}}))" >> $O/${T}_spec_bench.jsonl
done
echo done
