"""Fused-kernel time of a config under knob settings given as k=v[,k=v] groups:
python tools/knob_probe.py CONFIG 'prefetch=8' 'serp=1,prefetch=8' ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_19702_b200 import MIEngine, datagen
from paper_2411_19702_b200 import _native as nat

cfg = int(sys.argv[1])
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


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); t.append(a.elapsed_time(b))
    return sorted(t)[len(t) // 2]


for spec in ["default"] + sys.argv[2:]:
    kv = {} if spec == "default" else {k: int(v) for k, v in (x.split("=") for x in spec.split(","))}
    old = {k: nat.get_tuning(k) for k in kv}
    nat.set_tuning(**kv)
    ms = timed(lambda: eng.compute(prep, None, dt, tiles=tl, out=out, tile_major=True))
    nat.set_tuning(**old)
    print(f"config {cfg} {spec}: fused {ms:.3f} ms", flush=True)
