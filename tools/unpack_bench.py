"""Kernel 1 alone: time MIEngine.prepare (unpack + column stats) per config."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_19702_b200 import MIEngine, datagen

eng = MIEngine.get(0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=eng.device)
for cfg in [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "3").split(",")]:
    rec = datagen.config_recipe(cfg)
    n, m = rec["n"], rec["m"]
    w = datagen.generate_words_device(rec, eng.device)
    prep = eng.prepare(w, n, m)
    ref = prep.x.clone(), prep.colsum.clone()
    torch.cuda.synchronize()
    ms = []
    for _ in range(10):
        flush.fill_(1)
        del prep
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); prep = eng.prepare(w, n, m); e1.record(); e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    ok = torch.equal(prep.x, ref[0]) and torch.equal(prep.colsum, ref[1])
    ld, m_pad = eng.layout(n, m)
    byt = w.numel() * 8 + ld * m_pad
    avg = sum(ms) / len(ms)
    print(f"cfg{cfg} unpack avg {avg:.4f} ms min {min(ms):.4f} ms  {byt / avg / 1e6:.0f} GB/s  deterministic={ok}")
    del prep, ref, w
    torch.cuda.empty_cache()
