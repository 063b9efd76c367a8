"""PCIe D2H rate of 2-D (strided) copies vs one contiguous copy, pinned host
destination: the staged egress of mi_all_pairs_host copies column strips.
    python tools/d2h_2d.py"""
import torch
from cuda.bindings import runtime as rt

m = 10000
dev = torch.empty((m, m), dtype=torch.float64, device="cuda")
host = torch.empty((m, m), dtype=torch.float64, pin_memory=True)
st = torch.cuda.current_stream().cuda_stream
K = rt.cudaMemcpyKind.cudaMemcpyDeviceToHost


def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); best = min(best, a.elapsed_time(b))
    return best


pitch = m * 8
full = t(lambda: rt.cudaMemcpyAsync(host.data_ptr(), dev.data_ptr(), m * pitch, K, st))
print(f"contiguous 800 MB: {full:.2f} ms = {m * pitch / full / 1e6:.1f} GB/s")
for w in (10000, 5000, 2500, 1250, 625, 256):
    rows = m
    ms = t(lambda: rt.cudaMemcpy2DAsync(host.data_ptr(), pitch, dev.data_ptr(), pitch, w * 8, rows, K, st))
    print(f"2-D {rows} rows x {w * 8} B: {ms:.2f} ms = {rows * w * 8 / ms / 1e6:.1f} GB/s")

s2 = torch.cuda.Stream()
ev = torch.cuda.Event()


def two(w):
    half = m // 2
    ev.record(torch.cuda.current_stream())  # both copies start together
    s2.wait_event(ev)
    rt.cudaMemcpy2DAsync(host.data_ptr(), pitch, dev.data_ptr(), pitch, w * 8, half, K, st)
    rt.cudaMemcpy2DAsync(host.data_ptr() + half * pitch, pitch, dev.data_ptr() + half * pitch, pitch, w * 8,
                         m - half, K, s2.cuda_stream)
    e2 = torch.cuda.Event(); e2.record(s2); torch.cuda.current_stream().wait_event(e2)


for w in (10000, 2500):
    ms = t(lambda: two(w))
    print(f"2 streams 2-D {m} rows x {w * 8} B: {ms:.2f} ms = {m * w * 8 / ms / 1e6:.1f} GB/s")


def two1d():
    half = m * m // 2 * 8
    ev.record(torch.cuda.current_stream())
    s2.wait_event(ev)
    rt.cudaMemcpyAsync(host.data_ptr(), dev.data_ptr(), half, K, st)
    rt.cudaMemcpyAsync(host.data_ptr() + half, dev.data_ptr() + half, half, K, s2.cuda_stream)
    e2 = torch.cuda.Event(); e2.record(s2); torch.cuda.current_stream().wait_event(e2)


ms = t(two1d)
print(f"2 streams 1-D 800 MB: {ms:.2f} ms = {m * pitch / ms / 1e6:.1f} GB/s")
