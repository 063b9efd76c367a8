"""Fused-kernel time of a config under knob settings given as k=v[,k=v] groups:
python tools/knob_probe.py CONFIG 'prefetch=8' 'serp=1,prefetch=8' ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_19702_b200 import MIEngine, datagen
from paper_2411_19702_b200 import _native as nat

cfg = int(sys.argv[1])
eng = MIEngine.get(0)
rec = datagen.config_recipe(cfg)
n, m = rec["n"], rec["m"]
dt = torch.float32 if datagen.CONFIGS[cfg]["out"] == "float32" else torch.float64
w = datagen.generate_words_device(rec, eng.device)
prep = eng.prepare(w, n, m)
tl = eng.tiles(m)
ts = int(nat.lib().mi_tile_size())
out = torch.empty((tl.shape[0], ts, ts), dtype=dt, device=eng.device)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=eng.device)


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); t.append(a.elapsed_time(b))
    return sorted(t)[len(t) // 2]


def clock_mhz():
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        return pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    except Exception:
        return -1


# Round robin over the settings (ROUNDS passes, 3 launches each): a power-capped
# GPU slows down over the first seconds of load, so settings measured one after
# another are not comparable (the first one runs ~10% faster at config 4).
specs = ["default"] + sys.argv[2:]
rounds = int(os.environ.get("ROUNDS", "3"))
res = {sp: [] for sp in specs}
for r in range(rounds):
    for spec in specs:
        kv = {} if spec == "default" else {k: int(v) for k, v in (x.split("=") for x in spec.split(","))}
        old = {k: nat.get_tuning(k) for k in kv}
        nat.set_tuning(**kv)
        ms = timed(lambda: eng.compute(prep, None, dt, tiles=tl, out=out, tile_major=True), reps=3)
        nat.set_tuning(**old)
        res[spec].append(ms)
        print(f"  round {r} config {cfg} {spec}: fused {ms:.3f} ms (SM {clock_mhz()} MHz after)", flush=True)
for spec in specs:
    v = sorted(res[spec])
    print(f"config {cfg} {spec}: fused median {v[len(v) // 2]:.3f} ms, min {v[0]:.3f}", flush=True)
