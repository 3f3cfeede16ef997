import os, sys, time, torch
sys.path.insert(0, "/root/repo")
from paper_2302_05045_b200 import samo
torch.cuda.init()
def run(batch, i, o, ms, sk):
    os.environ["SAMO_DW_MS"] = str(ms); os.environ["SAMO_DW_SK"] = str(sk)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = (torch.rand((batch, i), device="cuda", generator=g) * 2 - 1).half()
    dy = (torch.rand((batch, o), device="cuda", generator=g) * 2 - 1).half()
    out = samo.dw_gemm(x, dy); torch.cuda.synchronize()
    ref = (x.float().t() @ dy.float())
    err = (out.float() - ref).abs().max().item()
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(10): samo.dw_gemm(x, dy)
    t1.record(); torch.cuda.synchronize()
    print(f"b{batch} {i}x{o} ms{ms} sk{sk}: maxerr {err:.3g} time {t0.elapsed_time(t1)/10*1e3:.1f} us", flush=True)
for (b, i, o) in [(4096, 2560, 2560)]:
    for ms in (1,):
        for sk in (0, 1):
            run(b, i, o, ms, sk)
