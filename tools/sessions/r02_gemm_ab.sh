#!/bin/bash
# GEMM epilogue + K123 launch-bound A/B: dW tests, bench_dw on the old tree
# (ab_h) and the current one, then ab3 on the step.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_dw.py tests/test_gpu_parity.py -x -q > $O/r02j_pytest.log 2>&1; echo "rc=$?" >> $O/r02j_pytest.log
for d in ab_h . ab_h .; do
  (cd $d && timeout 300 python tools/bench_dw.py --reps 20 2>&1 | sed "s|^|$d |") >> $O/r02j_dw.log
done
bash tools/ab3.sh ab_h . > /dev/null 2>&1; cp $O/ab3.log $O/r02j_ab3.log
echo done
