"""mi_unpermute alone: GB/s (read + write) at a given size and element size.
    python tools/unpermute_bench.py --m 50000 --esz 4 [--reps 5] [--ctas 1]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_19702_b200 import _native as nat

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=50000)
ap.add_argument("--esz", type=int, default=4)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--ctas", type=int, default=1)
a = ap.parse_args()
dt = torch.float32 if a.esz == 4 else torch.float64
src = torch.empty((a.m, a.m), dtype=dt, device="cuda").uniform_()
out = torch.empty_like(src)
inv = torch.randperm(a.m, device="cuda").to(torch.int32)
nat.set_tuning(unperm_ctas=a.ctas)
st = torch.cuda.current_stream().cuda_stream
f = lambda: nat.check(nat.lib().mi_unpermute(src.data_ptr(), a.m, out.data_ptr(), a.m, a.m, a.esz, inv.data_ptr(), st))
f(); torch.cuda.synchronize()
ts = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); f(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
ms = min(ts)
print(f"m={a.m} esz={a.esz} ctas={a.ctas}: {ms:.3f} ms, {2 * a.m * a.m * a.esz / ms / 1e6:.0f} GB/s")
