#!/bin/bash
# expand variants at N GPUs: HEAD (.), st.na stores (ab_x1), sector skip + st.na (ab_x2);
# local-group parity of ab_x2 first.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out
N=${N:-2}
(cd ab_x2 && timeout 600 python -m pytest tests/test_gpu_dp.py -q -x -k "local_group and (3-default or 8-default or push_sinks)" > ../$O/r02y_x2_pytest.log 2>&1; echo "rc=$?" >> ../$O/r02y_x2_pytest.log)
: > $O/r02y_expand_ab.log
for d in . ab_x1 ab_x2 . ab_x1 ab_x2; do
  (cd $d && timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29661 \
    bench.py --gpus $N --steps 20 --warmup 5 --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d', d['ms_per_step'], d.get('phases_ms') or d.get('pipeline_phases_ms'))") >> $O/r02y_expand_ab.log
done
echo done
