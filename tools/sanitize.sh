#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the hot-path
# kernels at test sizes: config-1/2 steps (K123 and K1|K23, eager and graph),
# empty/full layers, K0 prune, the tcgen05 dW GEMM (plain and fused-sink
# forms), and the peer-to-peer step in a one-GPU local group at G = 3 and 8
# (peer stores, signals, the TMA-fed shard kernel).  Logs under gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out
T=${TAG:-r02san}
SEL="tests/test_gpu_parity.py::test_model_step_golden tests/test_gpu_parity.py::test_config1_fc4096_vs_oracle
 tests/test_gpu_parity.py::test_model_step_empty_and_full_layers tests/test_gpu_parity.py::test_prune_golden
 tests/test_gpu_parity.py::test_prune_multi_layer_vs_oracle tests/test_gpu_dw.py::test_sink_dw_equals_unfused_gather
 tests/test_gpu_dw.py::test_dw_gemm_vs_reference tests/test_gpu_dw.py::test_sink_dw_many_tiles_equals_unfused"
DP="tests/test_gpu_dp.py::test_local_group_p2p_bit_exact"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 50 --target-processes all \
    python -m pytest $SEL -x -q -p no:cacheprovider > $O/${T}_${tool}_step.log 2>&1
  echo "rc=$?" >> $O/${T}_${tool}_step.log
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 50 --target-processes all \
    python -m pytest $DP -k "3-default or 8-default or TMA1" -x -q -p no:cacheprovider > $O/${T}_${tool}_p2p.log 2>&1
  echo "rc=$?" >> $O/${T}_${tool}_p2p.log
done
echo done
