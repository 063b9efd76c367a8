import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_19702_b200 import MIEngine, datagen
eng = MIEngine.get(0)
rec = datagen.config_recipe(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
n, m = rec["n"], rec["m"]
w = datagen.generate_words_device(rec, eng.device).cpu().pin_memory()
out = torch.empty((m, m), dtype=torch.float64, pin_memory=True)
for it in range(3):
    t = time.perf_counter()
    eng.all_pairs_host(w, n, m, None, torch.float64, host_out=out)
    print(f"iter {it}: {1e3*(time.perf_counter()-t):.2f} ms", file=sys.stderr)
