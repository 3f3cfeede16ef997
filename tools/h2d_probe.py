"""H2D copy throughput from pinned host memory: one copy vs the same bytes
split across several streams (copy engines).  1 GPU."""
import torch

n = 5_303_106_560 // 2  # GPT-2.7B dense fp16 gradients
host = torch.empty(n, dtype=torch.float16, pin_memory=True)
dev = torch.empty(n, dtype=torch.float16, device="cuda")
for ns in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = (n + ns - 1) // ns
    best = 1e9
    for _ in range(4):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i, s in enumerate(streams):
            s.wait_event(a)
            with torch.cuda.stream(s):
                dev[i * chunk:(i + 1) * chunk].copy_(host[i * chunk:(i + 1) * chunk], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"streams={ns}: {best:.2f} ms, {2 * n / best / 1e6:.1f} GB/s", flush=True)
