"""The sparse backend's input (per-column index lists) to MI: host to_dense
(binmat.to_dense-style dense uint8 matrix + pack_bits, what as_dense_words
does) against the device packing (MIEngine.from_sparse), and the whole
drop-in call.  python tools/sparse_ingest.py [N M density]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2411_19702_b200 import MIEngine, mi_all_pairs
from paper_2411_19702_b200.binmat import as_dense_words

n, m, d = (int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])) if len(sys.argv) > 3 else (100_000, 10_000, 0.01)
rng = np.random.default_rng(0)


class Sparse:
    def __init__(self, n, m, cols):
        self.n_rows, self.n_cols, self.col_indices = n, m, tuple(cols)


k = rng.binomial(n, d, size=m)
cols = [np.sort(rng.choice(n, size=int(c), replace=False)).astype(np.int64) for c in k]
sp = Sparse(n, m, cols)
eng = MIEngine.get(0)
eng.from_sparse(sp); torch.cuda.synchronize()
t0 = time.perf_counter(); w_host = as_dense_words(sp)[2]; t1 = time.perf_counter()
w_dev = eng.from_sparse(sp).cpu().numpy().view(np.uint64); t2 = time.perf_counter()
assert np.array_equal(w_host, w_dev)
mi_all_pairs(sp)
t3 = time.perf_counter(); mi_all_pairs(sp); t4 = time.perf_counter()
print(f"N={n:,} m={m:,} density {d} nnz={int(k.sum()):,}: host to_dense + pack {1e3 * (t1 - t0):.0f} ms, "
      f"device from_sparse (upload indices, pack, download words) {1e3 * (t2 - t1):.0f} ms, "
      f"drop-in mi_all_pairs(sparse) {1e3 * (t4 - t3):.0f} ms", flush=True)
