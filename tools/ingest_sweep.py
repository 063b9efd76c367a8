"""End-to-end mi_all_pairs_host time (pinned words in, pinned MI out) per
"ingest" setting: 0 = one upload + row-band egress, S = S-stage pipeline.
    python tools/ingest_sweep.py [--config 3] [--stages 0,1,2,4,8] [--reps 10]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_19702_b200 import MIEngine, datagen
from paper_2411_19702_b200 import _native as nat

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--stages", default="0,1,2,4,8")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
eng = MIEngine.get(0)
rec = datagen.config_recipe(a.config)
n, m = rec["n"], rec["m"]
dt = torch.float64 if datagen.CONFIGS[a.config]["out"] == "float64" else torch.float32
w = datagen.generate_words_device(rec, eng.device).cpu().pin_memory()
out = torch.empty((m, m), dtype=dt, pin_memory=True)
ref = None
for s in [int(x) for x in a.stages.split(",")]:
    nat.set_tuning(ingest=s)
    for _ in range(2):
        eng.all_pairs_host(w, n, m, None, dt, host_out=out)
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); eng.all_pairs_host(w, n, m, None, dt, host_out=out); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    if ref is None:
        ref = out.clone()
    same = bool(torch.equal(out, ref))
    print(json.dumps({"config": a.config, "ingest": s, "ms_avg": round(sum(ts) / len(ts), 3), "ms_min": round(min(ts), 3),
                      "same_as_first": same}), flush=True)
