"""The drop-in mi_all_pairs(BinaryMatrix) end to end (pageable numpy words in,
fresh float64 numpy matrix out) on a BASELINE config, wall clock per call.
    python tools/dropin_e2e.py [--config 3] [--calls 4]"""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2411_19702_b200 import BinaryMatrix, datagen, mi_all_pairs

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--calls", type=int, default=4)
a = ap.parse_args()
rec = datagen.config_recipe(a.config)
n, m = rec["n"], rec["m"]
w = datagen.generate_words_device(rec, 0).cpu().numpy().view(np.uint64)
bm = BinaryMatrix(n, m, w)
ref = None
for i in range(a.calls):
    t = time.perf_counter()
    r = mi_all_pairs(bm)
    dt = time.perf_counter() - t
    if ref is None:
        ref = r.values.copy()
    print(f"call {i}: {dt * 1e3:.1f} ms  same={np.array_equal(r.values, ref)}", flush=True)
    del r
