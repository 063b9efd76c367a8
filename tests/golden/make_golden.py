"""Generate the golden fixtures that pin the oracle to the REAL reference.

Run once in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the reference package ``mimatrix`` read-only from
/root/reference/pkg/src and records, for a fixed list of inputs, the
reference's own outputs on the hot path:

* ``column_sums``            (binmat.py:175-177)
* ``gram_ones``              (gram.py:56-65 -> _kernels.py:48-61)
* ``gram_complete_optimized``(gram.py:88-111)       -> g00 / g01
* ``mi_all_pairs`` dense     (engine.py:144-168) in exact / epsilon /
  no-diagonal configurations
* ``generate``               (datagen.py:58-73) streams, incl. the
  config-1 and config-3 datasets named in BASELINE.json

Small cases are stored in full; large ones as SHA-256 digests of the exact
integer arrays plus a seeded sample of MI entries and the MI checksum.
Nothing at test time reads /root/reference: the tests only read the files
written here (golden.npz, golden_meta.json).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT_DIR = Path(__file__).resolve().parent

FULL_LIMIT = 130  # store G / MI in full up to this many columns
N_SAMPLE = 4096


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF_SRC)
    import mimatrix  # noqa: F401  (the reference, read-only)
    from mimatrix.binmat import column_sums, from_bits, from_rows
    from mimatrix.datagen import GenSpec, generate
    from mimatrix.engine import EngineConfig, mi_all_pairs, mi_all_pairs_naive
    from mimatrix.gram import gram_from_dense, gram_ones

    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"reference": REF_SRC, "cases": {}, "datagen": {}}

    def record(name: str, mat, extra_cfgs=(), naive=False):
        words = mat.words
        v = column_sums(mat)
        g = gram_ones(mat)
        gs = gram_from_dense(mat)
        mi = mi_all_pairs(mat).values
        m = mat.n_cols
        case = {
            "n_rows": int(mat.n_rows),
            "n_cols": int(m),
            "g11_sha256": sha(g.astype(np.int64)),
            "g00_sha256": sha(gs.g00.astype(np.int64)),
            "g01_sha256": sha(gs.g01.astype(np.int64)),
            "mi_checksum": float(mi.sum()),
            "full": bool(m <= FULL_LIMIT),
            "variants": [],
        }
        arrays[f"{name}/words"] = words
        arrays[f"{name}/v"] = v.astype(np.uint64)
        if m <= FULL_LIMIT:
            arrays[f"{name}/g11"] = g.astype(np.int64)
            arrays[f"{name}/mi"] = mi
        else:
            rng = np.random.default_rng(12345)
            k = min(N_SAMPLE, m * m)
            ii = rng.integers(0, m, k)
            jj = rng.integers(0, m, k)
            # always include the diagonal corners and tile-boundary positions
            extra = np.array([0, m - 1, min(127, m - 1), min(128, m - 1),
                              min(255, m - 1), min(256, m - 1)], dtype=np.int64)
            ii = np.concatenate([ii, extra, extra[::-1], extra])
            jj = np.concatenate([jj, extra, extra, extra[::-1]])
            arrays[f"{name}/sample_i"] = ii.astype(np.int64)
            arrays[f"{name}/sample_j"] = jj.astype(np.int64)
            arrays[f"{name}/sample_mi"] = mi[ii, jj]
            arrays[f"{name}/sample_g11"] = g[ii, jj].astype(np.int64)
        for vname, cfg in extra_cfgs:
            vv = mi_all_pairs(mat, cfg).values
            key = f"{name}/mi_{vname}"
            if m <= FULL_LIMIT:
                arrays[key] = vv
            else:
                arrays[key] = vv[arrays[f"{name}/sample_i"], arrays[f"{name}/sample_j"]]
            case["variants"].append({"name": vname, "mode": cfg.mode,
                                     "epsilon": cfg.epsilon,
                                     "include_diagonal": cfg.include_diagonal,
                                     "checksum": float(vv.sum())})
        if naive and m <= 64:
            arrays[f"{name}/mi_naive"] = mi_all_pairs_naive(mat).values
        meta["cases"][name] = case
        print(f"  {name}: n={mat.n_rows} m={m} checksum={case['mi_checksum']:.6f}")

    eps_cfg = ("epsilon", EngineConfig(mode="epsilon", epsilon=1e-12))
    eps_big = ("epsilon_1e-3", EngineConfig(mode="epsilon", epsilon=1e-3))
    nodiag = ("nodiag", EngineConfig(include_diagonal=False))

    print("known-answer cases (reference tests' fixtures)")
    # test_gram.py / conftest.py:49-52
    record("fixture_3x2", from_rows([[1, 0], [0, 1], [1, 1]]), [eps_cfg, nodiag], naive=True)
    # test_engine.py:25,90-93
    record("golden_0011_0111", from_rows([[0, 0], [0, 1], [1, 1], [1, 1]]), naive=True)
    # test_acceptance.py:120-123
    record("balanced_identical", from_rows([[0, 0], [1, 1], [0, 0], [1, 1]]), naive=True)
    record("independent", from_rows([[0, 0], [0, 1], [1, 0], [1, 1]]), naive=True)
    # test_engine.py:36-41 (H(0.75) on the diagonal)
    record("h075", from_rows([[1], [1], [1], [0]]))
    # test_engine.py:142-150
    record("single_column", from_rows([[1], [0], [1]]))
    record("single_row", from_rows([[1, 0, 1]]))
    # test_binmat.py:92-99 bit layout; test_io.py:72-78 65 x 1 all ones
    b = np.zeros((65, 1), dtype=np.uint8)
    b[0, 0] = 1
    b[64, 0] = 1
    record("layout_rows_0_64", from_bits(b))
    record("ones_65x1", from_bits(np.ones((65, 1), dtype=np.uint8)))
    record("zeros_4x2", from_bits(np.zeros((4, 2), dtype=np.uint8)), [eps_cfg])
    record("ones_7x2", from_bits(np.ones((7, 2), dtype=np.uint8)), [eps_cfg])

    print("random cases (conftest.rand_bits recipe: default_rng(seed).random < d)")
    shapes = [
        (1, 1, 0.5, 1), (1, 64, 0.5, 2), (64, 1, 0.0, 3), (65, 2, 1.0, 4),
        (63, 3, 0.5, 5), (127, 7, 0.4, 6), (130, 10, 0.25, 43), (200, 30, 0.3, 31),
        (300, 20, 0.3, 42), (500, 64, 0.5, 2024), (128, 129, 0.3, 7),
        (129, 128, 0.7, 8), (250, 255, 0.5, 9), (257, 257, 0.05, 10),
        (1000, 300, 0.05, 11), (777, 300, 0.95, 12), (2049, 200, 0.5, 13),
        (4096, 513, 0.5, 14),
    ]
    for n, m, d, seed in shapes:
        rng = np.random.default_rng(seed)
        bits = (rng.random((n, m)) < d).astype(np.uint8)
        extras = [eps_cfg, eps_big, nodiag] if m in (20, 30, 64, 129, 300) else []
        record(f"rand_{n}x{m}_d{d}_s{seed}", from_bits(bits), extras, naive=(m <= 20))

    print("config 1 (BASELINE configs[0]): generate(GenSpec(1000, 500, 0.5, 0))")
    cfg1 = generate(GenSpec(1000, 500, 0.5, 0))
    record("cfg1_generate", cfg1)
    # SURVEY 8(d)1 planting: rng(0).choice(500, 4) -> 2 all-zero + 2 all-one columns
    bits = cfg1.to_bits()
    cols = np.random.default_rng(0).choice(500, 4, replace=False)
    bits[:, cols[0]] = 0
    bits[:, cols[1]] = 0
    bits[:, cols[2]] = 1
    bits[:, cols[3]] = 1
    meta["cfg1_planted_columns"] = [int(c) for c in cols]
    record("cfg1_planted", from_bits(bits), [eps_cfg, nodiag])

    print("datagen stream KATs (test_datagen.py:44-48)")
    for seed in (0, 1, 42, 2**63, 2**64 - 1):
        for dens in (0.0, 0.1, 0.5, 0.9, 1.0):
            key = f"gen_13x7_s{seed}_d{dens}"
            arrays[f"datagen/{key}"] = generate(GenSpec(13, 7, dens, seed)).words
    for (n, m, dens, seed) in [(100, 33, 0.3, 5), (64, 64, 0.5, 0), (65, 129, 0.25, 2**63 + 5)]:
        key = f"gen_{n}x{m}_s{seed}_d{dens}"
        arrays[f"datagen/{key}"] = generate(GenSpec(n, m, dens, seed)).words
    meta["datagen"]["cfg1"] = {"spec": [1000, 500, 0.5, 0], "words_sha256": sha(cfg1.words)}

    if os.environ.get("GOLDEN_SKIP_CFG3") != "1":
        print("config 3 stream digest: generate(GenSpec(100000, 10000, 0.5, 2)) (slow)")
        cfg3 = generate(GenSpec(100000, 10000, 0.5, 2))
        meta["datagen"]["cfg3"] = {
            "spec": [100000, 10000, 0.5, 2],
            "words_sha256": sha(cfg3.words),
            "colsum_sha256": sha(column_sums(cfg3).astype(np.uint64)),
            "words_head": [int(x) for x in cfg3.words[0, :4]],
            "words_tail": [int(x) for x in cfg3.words[-1, -4:]],
        }
        # a column subset through the reference engine (MI depends only on
        # the two columns and N), for parity at full N without the full matrix
        sub = np.random.default_rng(2).choice(10000, 300, replace=False)
        sub = np.unique(np.concatenate([sub, [0, 1, 255, 256, 511, 9999]]))
        from mimatrix.binmat import BinaryMatrix
        smat = BinaryMatrix(100000, len(sub), np.ascontiguousarray(cfg3.words[sub]))
        meta["cfg3_subset_columns"] = [int(c) for c in sub]
        record("cfg3_subset", smat)
        del cfg3

    np.savez_compressed(OUT_DIR / "golden.npz", **arrays)
    with open(OUT_DIR / "golden_meta.json", "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", OUT_DIR / "golden.npz", OUT_DIR / "golden_meta.json")


if __name__ == "__main__":
    main()
