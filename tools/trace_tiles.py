"""Per-tile timeline of cluster 0 (clock64): MMA issue window vs epilogue window."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_19702_b200 import MIEngine, datagen
from paper_2411_19702_b200 import _native as nat

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dt = {"f64": torch.float64, "f32": torch.float32, "i32": torch.int32}[sys.argv[2] if len(sys.argv) > 2 else "f64"]
eng = MIEngine.get(0)
rec = datagen.config_recipe(cfg)
n, m = rec["n"], rec["m"]
w = datagen.generate_words_device(rec, eng.device)
prep = eng.prepare(w, n, m)
out = torch.empty((m, m), dtype=dt, device=eng.device)
eng.compute(prep, None, dt, out=out)
tr = torch.zeros(64 * 4 + 256 * 4 + 64 * 4, dtype=torch.int64, device=eng.device)
nat.lib().mi_debug_set_trace.argtypes = [ctypes.c_void_p]
nat.lib().mi_debug_set_trace(tr.data_ptr())
eng.compute(prep, None, dt, out=out)
torch.cuda.synchronize()
nat.lib().mi_debug_set_trace(None)
allt = tr.cpu()
t = allt[:256].view(64, 4).tolist()
ct = allt[256:1280].view(256, 4)
ct = ct[ct[:, 0] != 0]
if len(ct):
    base = int(ct[:, 0].min())
    st, md, en = (ct[:, 0] - base) / 1e3, (ct[:, 1] - base) / 1e3, (ct[:, 2] - base) / 1e3
    print(f"clusters {len(ct)}: start spread {float(st.max()):.1f} us; main-done min/med/max "
          f"{float(md.min()):.1f}/{float(md.median()):.1f}/{float(md.max()):.1f} us; "
          f"end min/med/max {float(en.min()):.1f}/{float(en.median()):.1f}/{float(en.max()):.1f} us")
    order = torch.argsort(en, descending=True)[:8].tolist()
    print("  slowest clusters (id: main_done, end):", ", ".join(f"{i}: {float(md[i]):.0f}, {float(en[i]):.0f}" for i in order))
t0 = t[0][0]
print(f"cfg{cfg} {dt}: cycles relative to first MMA start (k = 1000 cycles)")
w = allt[1280:].view(64, 4).tolist()
print(" tile  mma_start mma_end(issue)  epi_start  epi_end   mma_len epi_len  mma_wait_for_acc  mma_wait_full  prod_wait_empty(r0,r1) prod_len")
for k, (a, b, c, d) in enumerate(t):
    if a == 0:
        break
    prev_end = t[k - 1][1] if k else a
    print(f"{k:5d} {(a-t0)/1e3:10.1f} {(b-t0)/1e3:10.1f} {(c-t0)/1e3:10.1f} {(d-t0)/1e3:9.1f} {(b-a)/1e3:8.1f} {(d-c)/1e3:7.1f} {(a-prev_end)/1e3:8.1f}"
          f" {w[k][0]/1e3:13.1f} {w[k][1]/1e3:10.1f} {w[k][2]/1e3:8.1f} {w[k][3]/1e3:9.1f}")
