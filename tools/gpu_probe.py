"""Quick GPU probe: counts + MI of one small random case vs the oracle.

Usage: python tools/gpu_probe.py [n] [m]   (MI_B200_CTA_GROUP=1 for the 1-SM variant)
"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle as O
from paper_2411_19702_b200 import MIEngine

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
m = int(sys.argv[2]) if len(sys.argv) > 2 else 300
rng = np.random.default_rng(1)
bits = (rng.random((n, m)) < 0.4).astype(np.uint8)
w = O.pack_bits(bits)
e = MIEngine.get(0)
t = time.time()
g, v = e.gram_counts(e.upload(w), n, m)
torch.cuda.synchronize()
g = g.cpu().numpy().astype(np.int64); v = v.cpu().numpy()
print("cg", os.environ.get("MI_B200_CTA_GROUP", "2"), "time", time.time() - t)
gr = O.c_gram_ones(w)
print("colsum ok", np.array_equal(v.astype(np.uint64), O.column_sums(w)))
bad = np.argwhere(g != gr)
print("G mismatches", len(bad), "of", m * m)
if len(bad):
    print("first", bad[:10].tolist(), g[tuple(bad[0])], gr[tuple(bad[0])])
    print("g[:4,:4]", g[:4, :4]); print("ref[:4,:4]", gr[:4, :4])
mi = e.all_pairs_device(e.upload(w), n, m).cpu().numpy()
ref = O.c_mi_all_pairs(w, n)
print("MI max err", np.abs(mi - ref).max(), "sym", np.array_equal(mi, mi.T))
bad = np.argwhere(mi != mi.T)
print("asymmetric elements:", len(bad))
if len(bad):
    for i, j in bad[:12]:
        print(i, j, repr(mi[i, j]), repr(mi[j, i]), repr(ref[i, j]), "tile", i // 256, j // 256)
    ii, jj = bad[:, 0], bad[:, 1]
    print("diag-tile fraction", np.mean(ii // 256 == jj // 256), "i<j fraction", np.mean(ii < jj))
