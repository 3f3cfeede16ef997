timeout 300 ncu --metrics gpu__time_duration.sum,l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg,gpc__cycles_elapsed.max,launch__cluster_dim_x,launch__grid_size,launch__block_size --clock-control none --csv python -c "
import torch
for (b,i,o) in [(4096,2560,10240),(4096,2560,2560)]:
    x=torch.randn(b,i,device='cuda').half(); dy=torch.randn(b,o,device='cuda').half()
    for _ in range(2): torch.matmul(x.t(),dy)
    from paper_2302_05045_b200 import samo
    for _ in range(2): samo.dw_gemm(x,dy)
torch.cuda.synchronize()
" > gpurun_out/cublas_ncu.csv 2>&1
