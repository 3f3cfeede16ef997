#!/bin/bash
# K23 / expand sector skipping: split-path parity (K1+K23), checked suite of the
# step tests, A/B of the split path against HEAD (ab_s), then (N GPUs) the DP tests.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_state.py -q -x > $O/r02t_pytest.log 2>&1; echo "rc=$?" >> $O/r02t_pytest.log
SAMO_LIB=$PWD/paper_2302_05045_b200/libsamo_cuda_checked.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dp.py -k "not two_gpus and not four and not three and not nccl" -q -x > $O/r02t_checked.log 2>&1; echo "rc=$?" >> $O/r02t_checked.log
SAMO_FUSED_STEP=0 bash tools/ab3.sh ab_s . > /dev/null 2>&1; cp $O/ab3.log $O/r02t_ab_split.log
echo done
