"""Fused-kernel time of a config under the debug masks that remove parts of
the epilogue (1: no stores, 2: no mirror stores, 4: no direct stores, 16: no
MMAs) -- what the epilogue costs the MMAs running beside it.
python tools/epi_probe.py [config] [debug,...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_19702_b200 import MIEngine, datagen
from paper_2411_19702_b200 import _native as nat

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
dbgs = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "0,1,2,4,16").split(",")]
eng = MIEngine.get(0)
rec = datagen.config_recipe(cfg)
n, m = rec["n"], rec["m"]
dt = torch.float32 if datagen.CONFIGS[cfg]["out"] == "float32" else torch.float64
w = datagen.generate_words_device(rec, eng.device)
prep = eng.prepare(w, n, m)
tl = eng.tiles(m)
ts = int(nat.lib().mi_tile_size())
out = torch.empty((tl.shape[0], ts, ts), dtype=dt, device=eng.device)  # tile-major, like the bench
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=eng.device)


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); t.append(a.elapsed_time(b))
    return sorted(t)[len(t) // 2]


for d in dbgs:
    nat.set_tuning(debug=d)
    ms = timed(lambda: eng.compute(prep, None, dt, tiles=tl, out=out, tile_major=True))
    print(f"config {cfg} debug {d}: fused {ms:.3f} ms", flush=True)
nat.set_tuning(debug=0)
