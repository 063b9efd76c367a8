"""PCIe H2D / D2H bandwidth with pinned host memory (CUDA events)."""
import torch
for nbytes in (125_040_000, 800_000_000):
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    for name, dst, src in (("H2D", d, h), ("D2H", h, d)):
        dst.copy_(src, non_blocking=True); torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); dst.copy_(src, non_blocking=True); b.record(); b.synchronize()
            ts.append(a.elapsed_time(b))
        ms = min(ts)
        print(f"{name} {nbytes/1e6:.0f} MB: {ms:.2f} ms  {nbytes/ms/1e6:.1f} GB/s")
