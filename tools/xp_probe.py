"""Fused-kernel time of the word-operand build against the unpack + TMA build
on tall-N / narrow-m shapes, with the debug masks that isolate data movement
(16: no MMAs) and the stores (1: compute, skip stores).
python tools/xp_probe.py [NxM ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import torch
from paper_2411_19702_b200 import MIEngine, datagen
from paper_2411_19702_b200 import _native as nat

eng = MIEngine.get(0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=eng.device)


def timed(fn, reps=7):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); best = min(best, a.elapsed_time(b))
    return best


shapes = [(8_000_000, 512), (4_000_000, 1024)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
for n, m in shapes:
    w = datagen.generate(n, m, 0.3, 11)
    out = torch.empty((m, m), dtype=torch.float64, device=eng.device)
    for xp in (0, 1):
        nat.set_tuning(xp=xp)
        prep = eng.prepare(w, n, m)
        row = []
        dbgs = [int(v) for v in os.environ.get("XP_DEBUGS", "0,16,1,48,80,112").split(",")] if xp else [0, 16]
        for dbg in dbgs:
            nat.set_tuning(debug=dbg)
            row.append(timed(lambda: eng.compute(prep, None, torch.float64, out=out)))
        nat.set_tuning(debug=0)
        print(f"N={n:,} m={m} xp={xp}: " + ", ".join(f"debug {d}: {t:.3f}" for d, t in zip(dbgs, row)),
              flush=True)
        del prep
    nat.set_tuning(xp=-1)

if os.environ.get("XP_TRACE"):
    # per-phase cycle sums of cluster 0 (gram_mi_sm100.cuh, XP builds)
    n, m = shapes[0]
    w = datagen.generate(n, m, 0.3, 11)
    out = torch.empty((m, m), dtype=torch.float64, device=eng.device)
    for dbg in [int(v) for v in os.environ.get("XP_DEBUGS", "0").split(",")]:
        nat.set_tuning(xp=1, debug=dbg)
        prep = eng.prepare(w, n, m)
        eng.compute(prep, None, torch.float64, out=out)
        tr = torch.zeros(4096, dtype=torch.int64, device=eng.device)
        nat.lib().mi_debug_set_trace.argtypes = [ctypes.c_void_p]
        nat.lib().mi_debug_set_trace(tr.data_ptr())
        eng.compute(prep, None, torch.float64, out=out)
        torch.cuda.synchronize()
        nat.lib().mi_debug_set_trace(None)
        x = tr[2048:2048 + 32].cpu().tolist()
        for r in (0, 1):
            b = x[8 * r: 8 * r + 6]
            k = max(b[5], 1)
            print(f"debug {dbg} rank {r}: k-blocks {b[5]}; cycles per k-block: raw wait {b[0] / k:.0f}, LDS {b[1] / k:.0f}, "
                  f"free-stage wait {b[2] / k:.0f}, expand+STS {b[3] / k:.0f}, fence+arrive {b[4] / k:.0f}; "
                  f"raw producer wait {x[24 + r] / k:.0f}")
        nat.set_tuning(debug=0)
