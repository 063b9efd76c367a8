"""Run the fused kernel of one config a few times (for ncu captures).

    python tools/fused_once.py CONFIG [f64|f32|i32] [REPS]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_19702_b200 import MIEngine, datagen

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
dt = {"f64": torch.float64, "f32": torch.float32, "i32": torch.int32}[sys.argv[2] if len(sys.argv) > 2 else "f32"]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
eng = MIEngine.get(0)
rec = datagen.config_recipe(cfg)
n, m = rec["n"], rec["m"]
w = datagen.generate_words_device(rec, eng.device)
prep = eng.prepare(w, n, m)
out = torch.empty((m, m), dtype=dt, device=eng.device)
for _ in range(reps):
    eng.compute(prep, None, dt, out=out)
torch.cuda.synchronize()
print("ok", cfg, dt, float(out[:4, :4].float().sum()))
