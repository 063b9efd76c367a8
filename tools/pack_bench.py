"""Device packing (MIEngine.pack_bits) throughput: uint8 (N, m) -> words,
against numpy's packbits path on the host (binmat.pack_bits, the reference's
from_bits algorithm) on a smaller slice.
    python tools/pack_bench.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2411_19702_b200 import MIEngine
from paper_2411_19702_b200.binmat import pack_bits

eng = MIEngine.get(0)
for n, m in ((100_000, 10_000), (50_000, 50_000), (100_000, 2_000)):
    bits = (torch.rand((n, m), device=eng.device) < 0.5).to(torch.uint8)
    eng.pack_bits(bits); torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); eng.pack_bits(bits, check=False); b.record(); b.synchronize(); best = min(best, a.elapsed_time(b))
    byt = n * m + m * ((n + 63) // 64) * 8
    print(f"device pack {n} x {m}: {best:.3f} ms  {byt / best / 1e6:.0f} GB/s")
    del bits
    torch.cuda.empty_cache()
h = (np.random.default_rng(0).random((100_000, 2_000)) < 0.5).astype(np.uint8)
t = time.perf_counter(); pack_bits(h); dt = time.perf_counter() - t
print(f"host numpy pack 100000 x 2000: {dt * 1e3:.1f} ms")
