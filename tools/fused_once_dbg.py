"""One config's fused launch (tile-major) under a debug mask, for ncu:
python tools/fused_once_dbg.py CONFIG DEBUG"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_19702_b200 import MIEngine, datagen
from paper_2411_19702_b200 import _native as nat

cfg, dbg = int(sys.argv[1]), int(sys.argv[2])
eng = MIEngine.get(0)
rec = datagen.config_recipe(cfg)
n, m = rec["n"], rec["m"]
dt = torch.float32 if datagen.CONFIGS[cfg]["out"] == "float32" else torch.float64
w = datagen.generate_words_device(rec, eng.device)
prep = eng.prepare(w, n, m)
tl = eng.tiles(m)
ts = int(nat.lib().mi_tile_size())
out = torch.empty((tl.shape[0], ts, ts), dtype=dt, device=eng.device)
nat.set_tuning(debug=dbg)
for _ in range(2):
    eng.compute(prep, None, dt, tiles=tl, out=out, tile_major=True)
torch.cuda.synchronize()
