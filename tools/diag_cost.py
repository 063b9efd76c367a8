"""Cost of diagonal tiles (I == J) against off-diagonal ones: the fused
kernel over the T diagonal tiles alone vs T off-diagonal tiles (I, I+1).
    python tools/diag_cost.py --configs 4,5"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2411_19702_b200 import MIEngine, datagen
from paper_2411_19702_b200 import _native as nat

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="4")
a = ap.parse_args()
eng = MIEngine.get(0)
for cfg in [int(x) for x in a.configs.split(",")]:
    rec = datagen.config_recipe(cfg)
    n, m = rec["n"], rec["m"]
    dt = torch.float64 if datagen.CONFIGS[cfg]["out"] == "float64" else torch.float32
    w = datagen.generate_words_device(rec, eng.device)
    out = torch.empty((m, m), dtype=dt, device=eng.device)
    prep = eng.prepare(w, n, m)
    T = -(-m // int(nat.lib().mi_tile_size()))
    k = (T - 1) // 74 * 74  # whole rounds only
    diag = torch.from_numpy(np.array([[i, i] for i in range(k)], dtype=np.int32)).to(eng.device)
    off = torch.from_numpy(np.array([[i, i + 1] for i in range(k)], dtype=np.int32)).to(eng.device)
    r = {"cfg": cfg, "tiles": k}
    for name, t in (("diag", diag), ("offdiag", off)):
        eng.compute(prep, None, dt, tiles=t, out=out); torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); eng.compute(prep, None, dt, tiles=t, out=out); e1.record(); e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        r[name + "_ms"] = round(best, 4)
    print(json.dumps(r), flush=True)
    del prep, out, w
    torch.cuda.empty_cache()
