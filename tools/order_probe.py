"""Column-sum order vs natural order, per config: fused kernel alone on each
order, the native ordered step (mi_column_order + ordered unpack + fused +
mi_unpermute) against the natural step (unpack + fused), and the pieces.

    python tools/order_probe.py --configs 2,4,5 [--unperm-ctas 1]
CUDA events, L2 flushed between repetitions.
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_19702_b200 import MIEngine, datagen
from paper_2411_19702_b200 import _native as nat

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="4")
ap.add_argument("--unperm-ctas", default="0")
a = ap.parse_args()
eng = MIEngine.get(0)
dev = eng.device
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)


def timed(fn, reps):
    fn(); torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    return sum(ms) / len(ms)


for cfg in [int(x) for x in a.configs.split(",")]:
    rec = datagen.config_recipe(cfg)
    n, m = rec["n"], rec["m"]
    dt = torch.float64 if datagen.CONFIGS[cfg]["out"] == "float64" else torch.float32
    reps = {1: 20, 2: 20, 3: 5, 4: 3, 5: 2}[cfg]
    w = datagen.generate_words_device(rec, dev)
    out = torch.empty((m, m), dtype=dt, device=dev)
    r = {"cfg": cfg, "auto": eng.choose_order(w, n, m)}
    prep = eng.prepare(w, n, m)
    r["natural_fused_ms"] = timed(lambda: eng.compute(prep, None, dt, out=out), reps)
    r["natural_step_ms"] = timed(lambda: eng.compute(eng.prepare(w, n, m), None, dt, out=out), reps)
    del prep
    torch.cuda.empty_cache()
    prep = eng.prepare(w, n, m, order="colsum")
    slot = torch.empty((m, m), dtype=dt, device=dev)
    tl = eng.tiles(m)
    st = torch.cuda.current_stream(dev).cuda_stream
    r["colsum_fused_ms"] = timed(lambda: nat.lib().mi_gram_mi(prep.x.data_ptr(), prep.colstat.data_ptr(), n, m,
                                                              prep.ld, 0, 1e-12, 1,
                                                              nat.MI_OUT_F64 if dt == torch.float64 else nat.MI_OUT_F32,
                                                              slot.data_ptr(), m, tl.data_ptr(), tl.shape[0], st), reps)
    r["column_order_ms"] = timed(lambda: eng.column_order(w, n, m), reps)
    for c in [int(x) for x in a.unperm_ctas.split(",")]:
        nat.set_tuning(unperm_ctas=c)
        r[f"unpermute_ms_ctas{c}"] = timed(lambda: nat.lib().mi_unpermute(slot.data_ptr(), m, out.data_ptr(), m, m,
                                                                          slot.element_size(), prep.inv.data_ptr(), st),
                                           reps)
    nat.set_tuning(unperm_ctas=0)
    del slot
    torch.cuda.empty_cache()
    r["colsum_step_ms"] = timed(lambda: eng.compute(eng.prepare(w, n, m, order="colsum"), None, dt, out=out), reps)
    r["unpermute_gbs"] = 2 * m * m * out.element_size() / (min(v for k, v in r.items() if k.startswith("unpermute_ms")) * 1e6)
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
    del prep, out, w
    torch.cuda.empty_cache()
