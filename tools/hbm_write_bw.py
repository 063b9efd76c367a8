"""Write-only and copy HBM bandwidth on this box (torch fill_/copy_, 1 GiB).

Caveat: torch's fill_ kernel reports ~3.9 TB/s of writes, well below what the
HBM takes; hand-written store kernels and cudaMemset reach 7.0-7.3 TB/s
(tools/micro/write_bw.cu), which is the write roofline DESIGN.md uses."""
import torch
x = torch.empty(1 << 30, dtype=torch.int8, device="cuda")
y = torch.empty(1 << 30, dtype=torch.int8, device="cuda")
for name, fn, nbytes in [("fill (write)", lambda: x.fill_(1), 1 << 30),
                         ("memset (write)", lambda: x.zero_(), 1 << 30),
                         ("copy (read+write)", lambda: y.copy_(x), 2 << 30)]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        fn()
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"{name}: {ms:.4f} ms  {nbytes / ms / 1e6:.0f} GB/s")
