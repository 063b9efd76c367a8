"""Every BASELINE config on one B200 with the current build: the step
(prepare + fused kernel, device-resident words, L2 flushed, median of 5) and
the fused kernel alone, as pair-samples/s and as a fraction of the tcgen05
peak measured on this GPU (mi_tensor_peak), with the operand path used.
python tools/config_table.py [configs]"""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_19702_b200 import MIEngine, datagen
from paper_2411_19702_b200 import _native as nat

eng = MIEngine.get(0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=eng.device)
peak = nat.tensor_peak(0, True, 0.05)["ops_per_s"]


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); t.append(a.elapsed_time(b))
    return statistics.median(t)


cfgs = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "1,2,3,4,5").split(",")]
for cfg in cfgs:
    rec = datagen.config_recipe(cfg)
    n, m = rec["n"], rec["m"]
    dt = torch.float64 if datagen.CONFIGS[cfg]["out"] == "float64" else torch.float32
    w = datagen.generate_words_device(rec, eng.device)
    tl = eng.tiles(m)
    ts = int(nat.lib().mi_tile_size())
    out = torch.empty((int(tl.shape[0]), ts, ts), dtype=dt, device=eng.device)
    W = n * m * (m + 1) / 2
    step = timed(lambda: eng.compute(eng.prepare(w, n, m), None, dt, tiles=tl, out=out, tile_major=True))
    prep = eng.prepare(w, n, m)
    eng.compute(prep, None, dt, tiles=tl, out=out, tile_major=True)  # statistics ready (word-operand path)
    fused = timed(lambda: eng.compute(prep, None, dt, tiles=tl, out=out, tile_major=True))
    print(json.dumps({"config": cfg, "N": n, "m": m, "out": str(dt).split(".")[-1],
                      "path": "words operand" if eng.words_operand(n, m) else "unpack + TMA",
                      "step_ms": round(step, 4), "fused_ms": round(fused, 4),
                      "pair_samples_per_s": W / (step * 1e-3),
                      "fused_frac_of_measured_peak": round(2 * W / (fused * 1e-3) / peak, 3),
                      "peak_pops": round(peak / 1e15, 3)}), flush=True)
    del w, out, prep
    torch.cuda.empty_cache()
