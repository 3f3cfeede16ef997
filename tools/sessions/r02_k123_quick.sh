#!/bin/bash
# Quick K123 check: step parity tests + the bench's K123 line (f16, bf16).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out
T=${TAG:-r02g}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $O/${T}_pytest.log 2>&1; echo "rc=$?" >> $O/${T}_pytest.log
for G in f16 bf16; do
timeout 300 python bench.py --profile --steps 20 --warmup 5 --grad-dtype $G 2>/dev/null | tail -1 | \
  python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']['K123_fused_step']; print(json.dumps({'grad':'$G','ms_step':d['ms_per_step'],'k123_ms':k['ms'],'GBps':k['GBps'],'frac':k['frac'],'k1':d['kernels']['K1_gather_unscale']['ms'],'k23':d['kernels']['K23_adam_downcast_expand']['ms']}))" >> $O/${T}_k123.jsonl
done
echo done
