"""Board power and SM clock of the fused kernel under sustained load, per debug
variant (what the 1 kW cap is spent on): back-to-back launches for SECONDS
each, NVML sampled every 5 ms.
    python tools/power_probe.py CONFIG [SECONDS] ['debug=16' 'debug=1' ...]"""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml
import torch
from paper_2411_19702_b200 import MIEngine, datagen
from paper_2411_19702_b200 import _native as nat

cfg = int(sys.argv[1])
seconds = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0
eng = MIEngine.get(0)
rec = datagen.config_recipe(cfg)
n, m = rec["n"], rec["m"]
dt = torch.float32 if datagen.CONFIGS[cfg]["out"] == "float32" else torch.float64
w = datagen.generate_words_device(rec, eng.device)
prep = eng.prepare(w, n, m)
tl = eng.tiles(m)
ts = int(nat.lib().mi_tile_size())
out = torch.empty((tl.shape[0], ts, ts), dtype=dt, device=eng.device)
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)


class Sampler(threading.Thread):
    def __init__(self):
        super().__init__(daemon=True)
        self.on, self.p, self.c = True, [], []

    def run(self):
        while self.on:
            self.p.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1e3)
            self.c.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            time.sleep(0.005)


def run(fn):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); fn(); b.record(); b.synchronize()
    reps = max(3, int(seconds * 1e3 / a.elapsed_time(b)))
    s = Sampler(); s.start()
    e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)  # mJ
    a.record()
    for _ in range(reps):
        fn()
    b.record(); b.synchronize()
    e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
    s.on = False; s.join()
    run.joules = (e1 - e0) / 1e3 / reps
    k = len(s.p) // 2  # second half: the controller has settled
    p2, c2 = s.p[k:], sorted(s.c[k:])
    return a.elapsed_time(b) / reps, sum(p2) / max(len(p2), 1), c2[len(c2) // 2] if c2 else -1


time.sleep(2.0)
print(f"idle: {pynvml.nvmlDeviceGetPowerUsage(h) / 1e3:.0f} W, SM {pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)} MHz")
for spec in ["default"] + sys.argv[3:]:
    kv = {} if spec == "default" else {k: int(v) for k, v in (x.split("=") for x in spec.split(","))}
    old = {k: nat.get_tuning(k) for k in kv}
    nat.set_tuning(**kv)
    ms, pw, mhz = run(lambda: eng.compute(prep, None, dt, tiles=tl, out=out, tile_major=True))
    nat.set_tuning(**old)
    print(f"config {cfg} {spec}: {ms:.3f} ms/launch, {pw:.0f} W, SM {mhz} MHz -> {ms * mhz * 1e3 / 1e6:.2f} Mcycles, {run.joules:.2f} J/launch", flush=True)
    time.sleep(3.0)
