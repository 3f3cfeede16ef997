#!/bin/bash
# Tensor-pipe activity and TMA bytes of our dW GEMM forms next to cuBLAS on
# MLP up, qkv and attn out (4096 tokens), one launch each after warm-up.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
cat > /tmp/dw_ncu.py <<'PY'
import torch, sys
sys.path.insert(0, ".")
from paper_2302_05045_b200 import samo
for (b, i, o) in [(4096, 2560, 10240), (4096, 2560, 7680), (4096, 2560, 2560)]:
    x = (torch.rand(b, i, device="cuda") * 2 - 1).half(); dy = (torch.rand(b, o, device="cuda") * 2 - 1).half()
    for _ in range(2): torch.matmul(x.t(), dy); samo.dw_gemm(x, dy)
    torch.cuda.synchronize()
PY
timeout 300 python /tmp/dw_ncu.py > gpurun_out/r02z_dw_ncu_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum,launch__grid_size,launch__cluster_dim_x \
  -k regex:"nvjet|k_dw_gemm" --clock-control none --csv python /tmp/dw_ncu.py > gpurun_out/r02z_dw_ncu.csv 2> gpurun_out/r02z_dw_ncu.err
echo "ncu rc=$?"
