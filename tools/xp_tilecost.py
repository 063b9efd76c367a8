"""Cost of one diagonal against one off-diagonal tile when a single tile is
split into K-range units over every SM pair, for both operand builds (the
weights of the K-range tail plan).
python tools/xp_tilecost.py [NxM ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
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


shapes = [(8_000_000, 512), (2_000_000, 1024)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
for n, m in shapes:
    w = datagen.generate(n, m, 0.3, 11)
    out = torch.empty((m, m), dtype=torch.float64, device=eng.device)
    T = -(-m // 256)
    lists = {"diag (0,0)": [(0, 0)], "off (0,1)": [(0, 1)], "diag x2": [(0, 0), (1, 1)],
             "all": [(i, j) for i in range(T) for j in range(i, T)]}
    for xp in (1, 0):
        nat.set_tuning(xp=xp)
        prep = eng.prepare(w, n, m)
        row = []
        for name, tl in lists.items():
            tiles = torch.tensor(np.array(tl, dtype=np.int32), device=eng.device)
            row.append((name, timed(lambda: eng.compute(prep, None, torch.float64, tiles=tiles, out=out))))
        print(f"N={n:,} m={m} xp={xp}: " + ", ".join(f"{k}: {t:.3f} ms" for k, t in row), flush=True)
        del prep
    nat.set_tuning(xp=-1)

# the whole triangle per diagonal-tile weight of the K-range plan (knob xp_diag_w)
ws = [int(v) for v in os.environ.get("XP_DIAG_W", "100,90,80,70,60").split(",")]
for n, m in shapes:
    w = datagen.generate(n, m, 0.3, 11)
    out = torch.empty((m, m), dtype=torch.float64, device=eng.device)
    nat.set_tuning(xp=1)
    prep = eng.prepare(w, n, m)
    row = []
    for dw in ws:
        nat.set_tuning(xp_diag_w=dw)
        row.append(timed(lambda: eng.compute(prep, None, torch.float64, out=out)))
    print(f"N={n:,} m={m} all tiles, xp_diag_w " + ", ".join(f"{d}: {t:.3f} ms" for d, t in zip(ws, row)), flush=True)
    nat.set_tuning(xp=-1, xp_diag_w=100)
    del prep
