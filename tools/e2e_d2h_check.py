"""Is the D2H inside mi_all_pairs_host slower than a standalone copy?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_19702_b200 import MIEngine, datagen
eng = MIEngine.get(0)
rec = datagen.config_recipe(3)
n, m = rec["n"], rec["m"]
w = datagen.generate_words_device(rec, eng.device).cpu().pin_memory()
out = torch.empty((m, m), dtype=torch.float64, pin_memory=True)
dev = torch.empty((m, m), dtype=torch.float64, device="cuda")
for it in range(3):
    t = time.perf_counter(); eng.all_pairs_host(w, n, m, None, torch.float64, host_out=out)
    e2e = time.perf_counter() - t
    torch.cuda.synchronize(); t = time.perf_counter(); out.copy_(dev, non_blocking=True); torch.cuda.synchronize()
    d2h = time.perf_counter() - t
    t = time.perf_counter(); dev.copy_(out, non_blocking=True); torch.cuda.synchronize()
    h2d = time.perf_counter() - t
    print(f"e2e {e2e*1e3:.2f} ms | standalone D2H 800 MB {d2h*1e3:.2f} ms ({8e8/d2h/1e9:.1f} GB/s) | H2D {h2d*1e3:.2f} ms")
