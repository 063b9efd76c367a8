"""Cost of cutting one rank's work into column-group stages (the staged
broadcast's compute side), measured at world 1 where the broadcasts vanish:
dispatch.mi_all_pairs_sharded(stages=S), CUDA events, L2 flushed.
    python tools/stage_overhead.py --configs 3,4 --stages 1,2,4"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_19702_b200 import MIEngine, datagen, dispatch

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="3,4")
ap.add_argument("--stages", default="1,2,4")
a = ap.parse_args()
eng = MIEngine.get(0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=eng.device)
for cfg in [int(x) for x in a.configs.split(",")]:
    rec = datagen.config_recipe(cfg)
    n, m = rec["n"], rec["m"]
    dt = torch.float64 if datagen.CONFIGS[cfg]["out"] == "float64" else torch.float32
    w = datagen.generate_words_device(rec, eng.device)
    out = torch.empty((m, m), dtype=dt, device=eng.device)
    ref = None
    for S in [int(x) for x in a.stages.split(",")]:
        f = lambda: dispatch.mi_all_pairs_sharded(eng, w, n, m, None, dt, out=out, stages=S)
        f(); torch.cuda.synchronize()
        ts = []
        for _ in range(5 if cfg <= 3 else 2):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); f(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
        if ref is None:
            ref = out.clone()
        print(json.dumps({"cfg": cfg, "stages": S, "ms": round(min(ts), 3), "same": bool(torch.equal(out, ref))}),
              flush=True)
    del out, ref, w
    torch.cuda.empty_cache()
