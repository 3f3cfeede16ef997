#!/bin/bash
# expand-pass sector skipping: local-group parity (normal + checked build),
# then on N GPUs the cross-process P2P tests and a bench A/B against ab_s.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out
N=${N:-2}
timeout 900 python -m pytest tests/test_gpu_dp.py tests/test_gpu_parity.py -q -x -k "local_group or step" > $O/r02u_pytest.log 2>&1; echo "rc=$?" >> $O/r02u_pytest.log
SAMO_LIB=$PWD/paper_2302_05045_b200/libsamo_cuda_checked.so timeout 900 python -m pytest tests/test_gpu_dp.py -q -x -k "local_group" > $O/r02u_checked.log 2>&1; echo "rc=$?" >> $O/r02u_checked.log
timeout 900 python -m pytest tests/test_gpu_dp.py -q -x -k "two_gpus and p2p" > $O/r02u_dp2.log 2>&1; echo "rc=$?" >> $O/r02u_dp2.log
: > $O/r02u_ab.log
for d in ab_s . ab_s .; do
  (cd $d && timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29651 \
    bench.py --gpus $N --steps 20 --warmup 5 --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d', d['ms_per_step'], d['phases_ms'])") >> $O/r02u_ab.log
done
echo done
