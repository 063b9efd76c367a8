"""Tuning sweep of the fused kernel: kernel time per (config, knob setting).

    python tools/sweep.py --configs 3,4,5 --prefetch 0,8,12 --l2hint 0,1 --band 8 [--cg 2]
Prints one JSON line per measurement (kernel-only CUDA-event time, L2 flushed).
"""
import argparse, itertools, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_19702_b200 import EngineConfig, MIEngine, datagen
from paper_2411_19702_b200 import _native as nat

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="3")
ap.add_argument("--prefetch", default="0")
ap.add_argument("--l2hint", default="1")
ap.add_argument("--band", default="8")
ap.add_argument("--cg", default="2")
ap.add_argument("--reps", type=int, default=0)
ap.add_argument("--stages", default="6")
ap.add_argument("--epi", default="8")
ap.add_argument("--dtype", default="auto")
ap.add_argument("--pace", default="-1")
ap.add_argument("--tail", default="1")
ap.add_argument("--fp4", default="1")
a = ap.parse_args()
ints = lambda s: [int(x) for x in s.split(",")]
eng = MIEngine.get(0)
dev = eng.device
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)
for cfg in ints(a.configs):
    rec = datagen.config_recipe(cfg)
    n, m = rec["n"], rec["m"]
    w = datagen.generate_words_device(rec, dev)
    prep, prep_ld = None, None
    dt = {"auto": torch.float64 if datagen.CONFIGS[cfg]["out"] == "float64" else torch.float32,
          "f64": torch.float64, "f32": torch.float32, "i32": torch.int32}[a.dtype]
    out = torch.empty((m, m), dtype=dt, device=dev)
    reps = a.reps or {1: 50, 2: 50, 3: 10, 4: 3, 5: 2}[cfg]
    W = n * m * (m + 1) / 2
    for cg, pf, hint, band, st, ew, pace, tail, fp4 in itertools.product(
            ints(a.cg), ints(a.prefetch), ints(a.l2hint), ints(a.band), ints(a.stages), ints(a.epi), ints(a.pace),
            ints(a.tail), ints(a.fp4)):
        nat.set_tuning(cta_group=cg, prefetch=pf, l2_hint=hint, band=band, stages=st, epi_warps=ew)
        for key, val in (("pace", pace), ("tail", tail), ("fp4", fp4)):  # newer knobs: absent from older A/B builds
            try:
                nat.set_tuning(**{key: val})
            except Exception:
                assert val == {"pace": -1, "tail": 1, "fp4": 0}[key], f"this build has no '{key}' knob"
        eng._tiles.clear()
        tiles = eng.tiles(m)
        if prep_ld != eng.layout(n, m):  # operand format follows the knobs (fp4, cta_group)
            prep = None
            torch.cuda.empty_cache()
            prep, prep_ld = eng.prepare(w, n, m), eng.layout(n, m)
        eng.compute(prep, None, dt, tiles=tiles, out=out)
        torch.cuda.synchronize()
        ms = []
        for _ in range(reps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); eng.compute(prep, None, dt, tiles=tiles, out=out); e1.record()
            e1.synchronize(); ms.append(e0.elapsed_time(e1))
        best, avg = min(ms), sum(ms) / len(ms)
        print(json.dumps({"cfg": cfg, "cg": cg, "prefetch": pf, "l2hint": hint, "band": band, "stages": st, "epi_warps": ew, "pace": pace, "tail": tail, "fp4": fp4, "dtype": str(dt).split(".")[-1],
                          "ms_avg": round(avg, 4), "ms_min": round(best, 4),
                          "tops_avg": round(2 * W / avg / 1e9, 1)}), flush=True)
    del prep, out, w
    torch.cuda.empty_cache()
