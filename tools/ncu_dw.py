"""Workload for the ncu capture of the dW GEMM (MLP-up shape, 4096 x 2560 x
10240, p = 0.9): three dense GEMMs and three fused sinks.

    python tools/ncu_dw.py             # run it bare first
    ncu --set full --import-source on --clock-control none -k regex:k_dw_gemm -c 2 \
        -o gpurun_out/dw python tools/ncu_dw.py
"""
import sys

import torch

sys.path.insert(0, '.')
from paper_2302_05045_b200 import samo  # noqa: E402

batch, n_in, n_out = 4096, 2560, 10240
x = (torch.rand(batch, n_in, device="cuda") * 2 - 1).half()
dy = ((torch.rand(batch, n_out, device="cuda") * 2 - 1) * 4).half()
n = n_in * n_out
idx = torch.randperm(n, device="cuda")[: n // 10].sort().values.to(torch.int32)
m = samo.SamoModel.from_index_sets([samo.PrunedIndexSet("fc.weight", n, idx)], [(n_in, n_out)], 0)
m.init_layer(0, torch.zeros(n, device="cuda"))
for _ in range(3):
    samo.dw_gemm(x, dy)
    m.sink_dw(0, x, dy)
torch.cuda.synchronize()
print("ok")
