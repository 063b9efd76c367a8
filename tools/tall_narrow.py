"""Tall-N / narrow-m shapes, where reading D dominates: the step (prepare +
fused kernel) on both operand paths -- the unpack + TMA path (xp = 0: kernel
1 writes X, the GEMM reads it back) and the word-operand path (xp = 1:
column statistics only, the GEMM's producer warps expand the words) -- with
algorithmic HBM rates (words read once, MI written).
python tools/tall_narrow.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_19702_b200 import MIEngine, datagen
from paper_2411_19702_b200 import _native as nat

eng = MIEngine.get(0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=eng.device)


def timed(fn, reps=7):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); best = min(best, a.elapsed_time(b))
    return best


shapes = [(8_000_000, 256), (8_000_000, 512), (4_000_000, 1024), (16_000_000, 256), (2_000_000, 2048),
          (1_000_000, 4096)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
for n, m in shapes:
    w = datagen.generate(n, m, 0.3, 11)
    out = torch.empty((m, m), dtype=torch.float64, device=eng.device)
    W = n * m * (m + 1) / 2
    words_b, mi_b = w.numel() * 8, m * m * 8
    res = {}
    for xp in (0, 1):
        nat.set_tuning(xp=xp)
        prep = eng.prepare(w, n, m)
        ref = eng.compute(prep, None, torch.float64, out=out).clone()
        t_p = timed(lambda: eng.prepare(w, n, m))
        t_f = timed(lambda: eng.compute(prep, None, torch.float64, out=out))
        t_s = timed(lambda: eng.compute(eng.prepare(w, n, m), None, torch.float64, out=out))
        res[xp] = (t_p, t_f, t_s, ref)
        del prep
    nat.set_tuning(xp=-1)
    same = torch.equal(res[0][3], res[1][3])
    for xp in (0, 1):
        t_p, t_f, t_s, _ = res[xp]
        print(f"N={n:>10,} m={m:>5} xp={xp}: prepare {t_p:.3f} ms, fused {t_f:.3f} ms "
              f"({2 * W / t_f / 1e9:.0f} TOP/s), step {t_s:.3f} ms = {W / (t_s * 1e-3):.3e} pair-samples/s, "
              f"{(words_b + mi_b) / t_s / 1e6:.0f} GB/s algorithmic (words + MI)", flush=True)
    print(f"    bit-identical: {same}", flush=True)
    del out, w
    torch.cuda.empty_cache()
