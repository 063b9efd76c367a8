"""Tall-N / narrow-m shapes, where reading D dominates: kernel 1 (unpack) and
the fused kernel timed separately, with their HBM rates (algorithmic bytes:
words read + X written for the unpack; X read + MI written for the fused
kernel).  python tools/tall_narrow.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_19702_b200 import MIEngine, datagen

eng = MIEngine.get(0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=eng.device)


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); best = min(best, a.elapsed_time(b))
    return best


for n, m in ((8_000_000, 256), (8_000_000, 512), (4_000_000, 1024), (16_000_000, 256)):
    w = datagen.generate(n, m, 0.3, 11)
    ld, m_pad = eng.layout(n, m)
    prep = eng.prepare(w, n, m)
    out = torch.empty((m, m), dtype=torch.float64, device=eng.device)
    t_u = timed(lambda: eng.prepare(w, n, m))
    t_f = timed(lambda: eng.compute(prep, None, torch.float64, out=out))
    words_b, x_b, mi_b = w.numel() * 8, ld * m_pad, m * m * 8
    W = n * m * (m + 1) / 2
    print(f"N={n:>10,} m={m:>5}: unpack {t_u:.3f} ms ({(words_b + x_b) / t_u / 1e6:.0f} GB/s), "
          f"fused {t_f:.3f} ms ({(x_b + mi_b) / t_f / 1e6:.0f} GB/s of X + MI, "
          f"{2 * W / t_f / 1e9:.0f} TOP/s), step {W / ((t_u + t_f) * 1e-3):.3e} pair-samples/s", flush=True)
    del prep, out, w
    torch.cuda.empty_cache()
