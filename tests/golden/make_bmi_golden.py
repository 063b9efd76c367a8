"""Golden BMI1 containers written by the REAL reference's io.write_bmi.

Run once in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_bmi_golden.py

Writes tests/golden/bmi/*.bmi (valid files from write_bmi, io.py:85-89) plus
the malformed variants the reference's own tests construct
(test_io.py:87-111: bad magic, truncated payload, nonzero padding bits), and
bmi_meta.json with each valid file's shape and column sums
(binmat.column_sums, binmat.py:175-177).  Tests read only these files.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from mimatrix.binmat import column_sums, from_bits, from_rows  # noqa: E402
from mimatrix.io import read_bmi, write_bmi  # noqa: E402

OUT = Path(__file__).resolve().parent / "bmi"
OUT.mkdir(exist_ok=True)

cases = {
    "fixture_3x2": from_rows([[1, 0], [1, 1], [0, 1]]),
    "pad_65x5": from_bits((np.random.default_rng(5).random((65, 5)) < 0.5).astype(np.uint8)),
    "rand_1000x300": from_bits((np.random.default_rng(7).random((1000, 300)) < 0.3).astype(np.uint8)),
    "one_1x1": from_rows([[1]]),
}
meta = {}
for name, mat in cases.items():
    p = OUT / f"{name}.bmi"
    write_bmi(mat, p)
    assert read_bmi(p) == mat
    meta[name] = {"n_rows": mat.n_rows, "n_cols": mat.n_cols,
                  "column_sums": [int(x) for x in column_sums(mat)]}

# malformed files, built the way the reference's tests build them
raw = (OUT / "fixture_3x2.bmi").read_bytes()
(OUT / "bad_magic.bmi").write_bytes(b"XMI1" + raw[4:])
(OUT / "truncated.bmi").write_bytes(raw[:-8])
(OUT / "short_header.bmi").write_bytes(raw[:10])
pad = bytearray((OUT / "fixture_3x2.bmi").read_bytes())
pad[20] |= 0x80  # bit 7 of column 0's only word: row 7 of a 3-row matrix
(OUT / "dirty_padding.bmi").write_bytes(bytes(pad))
(OUT / "bmi_meta.json").write_text(json.dumps(meta, indent=1))
print("wrote", sorted(x.name for x in OUT.iterdir()))
