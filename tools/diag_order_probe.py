"""Config-4 fused-kernel time with the diagonal tiles moved out of the banded
order (first / last): their epilogue is slower than a tile's MMAs, and a pair
held up by one holds every pair up through the L2 pacing window.
    python tools/diag_order_probe.py [CONFIG]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_19702_b200 import MIEngine, datagen
from paper_2411_19702_b200 import _native as nat

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
eng = MIEngine.get(0)
rec = datagen.config_recipe(cfg)
n, m = rec["n"], rec["m"]
dt = torch.float32 if datagen.CONFIGS[cfg]["out"] == "float32" else torch.float64
w = datagen.generate_words_device(rec, eng.device)
prep = eng.prepare(w, n, m)
tl = eng.tiles(m)
ts = int(nat.lib().mi_tile_size())
out = torch.empty((tl.shape[0], ts, ts), dtype=dt, device=eng.device)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=eng.device)
d = tl[:, 0] == tl[:, 1]
orders = {"banded": tl, "diag first": torch.cat([tl[d], tl[~d]]).contiguous(), "diag last": torch.cat([tl[~d], tl[d]]).contiguous()}


def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); t.append(a.elapsed_time(b))
    return sorted(t)[len(t) // 2]


import time


def sustained(fn, seconds=2.0):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); fn(); b.record(); b.synchronize()
    reps = max(3, int(seconds * 1e3 / a.elapsed_time(b)))
    a.record()
    for _ in range(reps):
        fn()
    b.record(); b.synchronize()
    return a.elapsed_time(b) / reps


# sustained (2 s back to back per order, alternating): on a power-capped GPU
# only long windows compare to ~0.1%
for r in range(int(os.environ.get("ROUNDS", "2"))):
    for k, t in orders.items():
        ms = sustained(lambda: eng.compute(prep, None, dt, tiles=t, out=out, tile_major=True))
        print(f"config {cfg} {k}: sustained {ms:.3f} ms/launch", flush=True)
        time.sleep(2.0)
