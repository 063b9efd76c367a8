"""float32 epilogue (f32_epi) against the float64 path on full BASELINE configs.

    python tools/f32_epi_check.py --configs 2,4 [--reps 3]
For each config: fused-kernel time with f32_epi = 1 (FP32-pipe epilogue) and
0 (FP64 epilogue), and max |MI_f32 - MI_f64| over the whole matrix, where
MI_f64 is the float64-output result (within 1e-12 of the reference).
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_19702_b200 import MIEngine, datagen
from paper_2411_19702_b200 import _native as nat

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="2,4")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
eng = MIEngine.get(0)
dev = eng.device
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)
for cfg in [int(x) for x in a.configs.split(",")]:
    rec = datagen.config_recipe(cfg)
    n, m = rec["n"], rec["m"]
    w = datagen.generate_words_device(rec, dev)
    prep = eng.prepare(w, n, m)
    ref = eng.compute(prep, None, torch.float64)
    out = torch.empty((m, m), dtype=torch.float32, device=dev)
    res = {"config": cfg, "n": n, "m": m}
    for f32 in (1, 0):
        nat.set_tuning(f32_epi=f32)
        eng.compute(prep, None, torch.float32, out=out)
        torch.cuda.synchronize()
        ms = []
        for _ in range(a.reps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            eng.compute(prep, None, torch.float32, out=out)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        err = 0.0
        for r0 in range(0, m, 4096):
            d = (out[r0:r0 + 4096].double() - ref[r0:r0 + 4096]).abs().max().item()
            err = max(err, d)
        sym = bool(torch.equal(out, out.t()))
        res[f"f32_epi={f32}"] = {"ms": min(ms), "ms_all": ms, "max_abs_vs_f64": err, "symmetric": sym}
    nat.set_tuning(f32_epi=1)
    print(json.dumps(res), flush=True)
    del ref, out, prep
    torch.cuda.empty_cache()
