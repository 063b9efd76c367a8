"""CPU ORACLE -- test infrastructure only.

This module restates, in NumPy, the reference's algorithm for the hot path
(arxiv 2411.19702, package ``mimatrix``) so that the CUDA engine can be
checked against it.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline / ``--impl reference`` leg may import it, and
only as the checker or the timed CPU baseline -- never as a product path.
The product (``paper_2411_19702_b200``) never imports anything from here.

Pinned: every function is checked against the real reference's outputs
(``tests/golden/golden.npz``, produced by ``tests/golden/make_golden.py``,
which imports /root/reference) in ``tests/test_oracle.py``.

Citations are ``path:line`` relative to /root/reference/pkg/src/mimatrix/.
"""

from __future__ import annotations

import ctypes
import math
import os
from pathlib import Path

import numpy as np

WORD_BITS = 64
MODES = ("exact", "epsilon")

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "libmi_oracle.so"


class OracleError(Exception):
    """Raised for inconsistent inputs (mirrors errors.ConsistencyError)."""


# ----------------------------------------------------------------------------
# data model  (binmat.py)
# ----------------------------------------------------------------------------

def n_words(n_rows: int) -> int:
    """binmat.py:21-22"""
    return (n_rows + WORD_BITS - 1) // WORD_BITS


def pad_mask(n_rows: int) -> int:
    """binmat.py:25-30 -- valid bits of the last word of a column."""
    rem = n_rows % WORD_BITS
    return (1 << 64) - 1 if rem == 0 else (1 << rem) - 1


def pack_bits(bits: np.ndarray) -> np.ndarray:
    """binmat.py:34-46 -- (n, m) {0,1} -> (m, nw) uint64, bit r of word w = row 64w+r."""
    n, m = bits.shape
    nw = n_words(n)
    padded = np.zeros((m, nw * WORD_BITS), dtype=np.uint8)
    padded[:, :n] = bits.T
    packed = np.packbits(padded, axis=1, bitorder="little")
    return np.ascontiguousarray(packed).view("<u8").astype(np.uint64, copy=False).reshape(m, nw)


def unpack_bits(words: np.ndarray, n_rows: int) -> np.ndarray:
    """binmat.py:49-54"""
    m, nw = words.shape
    as_bytes = words.astype("<u8").view(np.uint8).reshape(m, nw * 8)
    bits = np.unpackbits(as_bytes, axis=1, bitorder="little", count=n_rows)
    return np.ascontiguousarray(bits.T)


def column_sums(words: np.ndarray) -> np.ndarray:
    """binmat.py:175-177 -- popcount of every word, summed per column."""
    return np.bitwise_count(words).sum(axis=1, dtype=np.uint64)


# ----------------------------------------------------------------------------
# counting  (gram.py, _kernels.py)
# ----------------------------------------------------------------------------

def gram_ones(words: np.ndarray, row_block: int = 64) -> np.ndarray:
    """_kernels.py:36-61 -- G11[i,j] = sum_w popcount(w_i & w_j), both triangles.

    Same AND + popcount algorithm as the numba kernel, vectorised over a
    block of rows at a time instead of prange over paired rows.
    """
    words = np.ascontiguousarray(words, dtype=np.uint64)
    m = words.shape[0]
    out = np.zeros((m, m), dtype=np.int64)
    for i0 in range(0, m, row_block):
        blk = words[i0:i0 + row_block]
        cnt = np.bitwise_count(blk[:, None, :] & words[None, :, :]).sum(axis=2, dtype=np.int64)
        out[i0:i0 + row_block] = cnt
    return out


def gram_complete_optimized(g11: np.ndarray, v: np.ndarray, n: int):
    """gram.py:88-111 -- closed-form g00/g01 with the reference's checks."""
    g11 = np.asarray(g11, dtype=np.int64)
    v = np.asarray(v, dtype=np.uint64)
    if not np.array_equal(g11, g11.T):
        raise OracleError("g11 must be symmetric")
    vi = v.astype(np.int64)
    if not np.array_equal(np.diagonal(g11), vi):
        raise OracleError("diagonal of g11 must equal the column sums")
    if np.any(vi > n) or np.any(vi < 0):
        raise OracleError(f"column sums must lie in [0, {n}]")
    g00 = (n + g11) - vi[:, None] - vi[None, :]
    g01 = vi[None, :] - g11
    for name, mat in (("g11", g11), ("g00", g00), ("g01", g01)):
        if mat.min(initial=0) < 0 or mat.max(initial=0) > n:
            raise OracleError(f"{name} entry outside [0, {n}]")
    return g11, g00, g01


# ----------------------------------------------------------------------------
# MI assembly  (engine.py)
# ----------------------------------------------------------------------------

def _term_exact(p, e):
    """engine.py:105-109"""
    with np.errstate(divide="ignore", invalid="ignore"):
        t = p * np.log2(p / e)
    return np.where(p > 0.0, t, 0.0)


def _term_epsilon(p, e, eps):
    """engine.py:112-113"""
    return p * np.log2((p + eps) / (e + eps))


def mi_from_counts(g11, g00, g01, n, mode="exact", epsilon=1e-12, include_diagonal=True):
    """engine.py:93-102 (probabilities) + engine.py:116-141 (mi_from_probabilities).

    Cells in the fixed order (1,1), (1,0), (0,1), (0,0); upper triangle
    mirrored; optional zero diagonal.
    """
    nf = float(n)
    p11 = g11 / nf
    p00 = g00 / nf
    p01 = g01 / nf
    p1 = np.diagonal(g11) / nf
    p0 = np.diagonal(g00) / nf
    cells = (
        (p11, np.outer(p1, p1)),
        (p01.T, np.outer(p1, p0)),
        (p01, np.outer(p0, p1)),
        (p00, np.outer(p0, p0)),
    )
    m = p1.shape[0]
    mi = np.zeros((m, m), dtype=np.float64)
    for joint, expected in cells:
        if mode == "exact":
            mi += _term_exact(joint, expected)
        else:
            mi += _term_epsilon(joint, expected, epsilon)
    mi = np.triu(mi) + np.triu(mi, 1).T
    if not include_diagonal:
        np.fill_diagonal(mi, 0.0)
    return mi


def mi_all_pairs(words: np.ndarray, n_rows: int, mode="exact", epsilon=1e-12,
                 include_diagonal=True) -> np.ndarray:
    """engine.py:144-168 with backend="dense": gram_ones -> column_sums ->
    gram_complete_optimized -> probabilities -> mi_from_probabilities."""
    g11 = gram_ones(words)
    v = column_sums(words)
    g11, g00, g01 = gram_complete_optimized(g11, v, n_rows)
    return mi_from_counts(g11, g00, g01, n_rows, mode, epsilon, include_diagonal)


def binary_entropy(p1: float) -> float:
    """engine.py:81-90"""
    h = 0.0
    if p1 > 0.0:
        h -= p1 * math.log2(p1)
    if p1 < 1.0:
        h -= (1.0 - p1) * math.log2(1.0 - p1)
    return h


def mi_pairwise_naive(x, y) -> float:
    """engine.py:171-202,205-220 -- direct four-cell count, exact mode."""
    xb = np.asarray(x).astype(bool)
    yb = np.asarray(y).astype(bool)
    n = xb.shape[0]
    c11 = int(np.count_nonzero(xb & yb))
    c10 = int(np.count_nonzero(xb & ~yb))
    c01 = int(np.count_nonzero(~xb & yb))
    c00 = int(np.count_nonzero(~xb & ~yb))
    px1 = (c11 + c10) / n
    px0 = (c01 + c00) / n
    py1 = (c11 + c01) / n
    py0 = (c10 + c00) / n
    total = 0.0
    for joint, expected in ((c11 / n, px1 * py1), (c10 / n, px1 * py0),
                            (c01 / n, px0 * py1), (c00 / n, px0 * py0)):
        if joint > 0.0:
            total += joint * math.log2(joint / expected)
    return total


# ----------------------------------------------------------------------------
# synthetic data  (datagen.py) + the BASELINE config recipes
# ----------------------------------------------------------------------------

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)
FLIP_SEED_XOR = 0xA5A5A5A5A5A5A5A5


def splitmix64_block(seed: int, start: int, count: int) -> np.ndarray:
    """datagen.py:44-50 -- draw k uses state seed + k*gamma."""
    idx = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + idx * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _MIX1
        z = (z ^ (z >> np.uint64(27))) * _MIX2
    return z ^ (z >> np.uint64(31))


def threshold(density: float) -> int:
    """datagen.py:53-55 -- smallest t with (draw < t) == (draw/2^64 < density)."""
    return math.ceil(density * (1 << 64))


def generate_bits(n: int, m: int, density, seed: int) -> np.ndarray:
    """datagen.py:58-73 -- row-major draws starting at index 1.

    ``density`` may be a scalar (the reference's GenSpec) or a length-m
    array of per-column densities (the BASELINE config recipes).
    """
    dens = np.broadcast_to(np.asarray(density, dtype=np.float64), (m,))
    thr = [threshold(float(d)) for d in dens]
    draws = splitmix64_block(seed, 1, n * m).reshape(n, m)
    bits = np.empty((n, m), dtype=np.uint8)
    for c in range(m):
        t = thr[c]
        if t <= 0:
            bits[:, c] = 0
        elif t >= 1 << 64:
            bits[:, c] = 1
        else:
            bits[:, c] = draws[:, c] < np.uint64(t)
    return bits


def config_recipe(cfg: int, n: int | None = None, m: int | None = None) -> dict:
    """per-column densities and planting for the 5 configs.

    Returns {n, m, seed, density (m,), zero_cols, one_cols, pairs (src, dst),
    flip_density}.  ``n``/``m`` may be overridden to get a small instance of
    the same recipe.
    """
    base = {1: (1000, 500, 0), 2: (10000, 2000, 1), 3: (100000, 10000, 2),
            4: (50000, 50000, 3), 5: (1000000, 20000, 4)}[cfg]
    n = base[0] if n is None else n
    m = base[1] if m is None else m
    seed = base[2]
    rng = np.random.default_rng(seed)
    out = {"n": n, "m": m, "seed": seed, "zero_cols": [], "one_cols": [],
           "pairs": [], "flip_density": 0.0}
    if cfg in (1, 3):
        out["density"] = np.full(m, 0.5)
        if cfg == 1:
            cols = rng.choice(m, 4, replace=False)
            out["zero_cols"] = [int(cols[0]), int(cols[1])]
            out["one_cols"] = [int(cols[2]), int(cols[3])]
    elif cfg == 2:
        out["density"] = rng.uniform(0.05, 0.95, m)
        k = min(200, m // 2)
        cols = rng.choice(m, 2 * k, replace=False)
        out["pairs"] = [(int(s), int(t)) for s, t in zip(cols[:k], cols[k:])]
        out["flip_density"] = 0.1
    elif cfg == 4:
        out["density"] = rng.beta(0.5, 20.0, m)
        k = max(1, m // 100)
        targets = rng.choice(m, k, replace=False)
        tset = set(int(t) for t in targets)
        pool = np.array([c for c in range(m) if c not in tset])
        sources = rng.choice(pool, k, replace=True)
        out["pairs"] = [(int(s), int(t)) for s, t in zip(sources, targets)]
        out["flip_density"] = 0.05
    elif cfg == 5:
        out["density"] = rng.uniform(0.01, 0.99, m)
    return out


def generate_config_bits(recipe: dict) -> np.ndarray:
    """Bits of a config recipe: base stream, constant columns, planted noisy copies.

    Flip bits come from the same splitmix64 stream with seed ^ 0xA5A5...A5,
    at the same cell index as the target cell.
    """
    n, m, seed = recipe["n"], recipe["m"], recipe["seed"]
    bits = generate_bits(n, m, recipe["density"], seed)
    for c in recipe["zero_cols"]:
        bits[:, c] = 0
    for c in recipe["one_cols"]:
        bits[:, c] = 1
    if recipe["pairs"]:
        flips = generate_bits(n, m, recipe["flip_density"], seed ^ FLIP_SEED_XOR)
        for s, t in recipe["pairs"]:
            bits[:, t] = bits[:, s] ^ flips[:, t]
    return bits


def generate_config_columns(recipe: dict, cols) -> np.ndarray:
    """Bits (n, len(cols)) of only the listed columns of a config recipe.

    Same values as generate_config_bits(recipe)[:, cols], without drawing the
    other m - len(cols) columns (draw index r*m + c + 1 is computed per column),
    so a bounded CPU baseline can use full-N column subsets of big configs.
    """
    n, m, seed = recipe["n"], recipe["m"], recipe["seed"]
    cols = [int(c) for c in cols]
    dens = np.broadcast_to(np.asarray(recipe["density"], dtype=np.float64), (m,))
    zero, one = set(recipe["zero_cols"]), set(recipe["one_cols"])
    src_of = {t: s for s, t in recipe["pairs"]}
    rows = np.arange(n, dtype=np.uint64)

    def base(c):
        t = threshold(float(dens[c]))
        if t <= 0:
            return np.zeros(n, dtype=np.uint8)
        if t >= 1 << 64:
            return np.ones(n, dtype=np.uint8)
        with np.errstate(over="ignore"):
            idx = rows * np.uint64(m) + np.uint64(c + 1)
            z = np.uint64(seed) + idx * _GAMMA
            z = (z ^ (z >> np.uint64(30))) * _MIX1
            z = (z ^ (z >> np.uint64(27))) * _MIX2
            z = z ^ (z >> np.uint64(31))
        return (z < np.uint64(t)).astype(np.uint8)

    def flip(c):
        t = threshold(recipe["flip_density"])
        with np.errstate(over="ignore"):
            idx = rows * np.uint64(m) + np.uint64(c + 1)
            z = np.uint64(seed ^ FLIP_SEED_XOR) + idx * _GAMMA
            z = (z ^ (z >> np.uint64(30))) * _MIX1
            z = (z ^ (z >> np.uint64(27))) * _MIX2
            z = z ^ (z >> np.uint64(31))
        return (z < np.uint64(min(t, (1 << 64) - 1))).astype(np.uint8)

    out = np.empty((n, len(cols)), dtype=np.uint8)
    for k, c in enumerate(cols):
        if c in zero:
            out[:, k] = 0
        elif c in one:
            out[:, k] = 1
        elif c in src_of:
            out[:, k] = base(src_of[c]) ^ flip(c)
        else:
            out[:, k] = base(c)
    return out


# ----------------------------------------------------------------------------
# the C restatement (oracle/mi_oracle.c), for sizes the NumPy path is too slow for
# ----------------------------------------------------------------------------

_lib = None


def c_lib():
    """Load oracle/_build/libmi_oracle.so (built by ``make -C oracle``)."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise OracleError(f"{_LIB_PATH} missing: run `make -C oracle`")
        lib = ctypes.CDLL(str(_LIB_PATH))
        u64p = ctypes.POINTER(ctypes.c_uint64)
        i64p = ctypes.POINTER(ctypes.c_int64)
        f64p = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        lib.oracle_column_sums.argtypes = [u64p, i64, i64, u64p]
        lib.oracle_gram_ones.argtypes = [u64p, i64, i64, i64p]
        lib.oracle_mi_all_pairs.argtypes = [u64p, i64, i64, i64, ctypes.c_int,
                                            ctypes.c_double, ctypes.c_int, f64p]
        lib.oracle_mi_all_pairs.restype = ctypes.c_int
        lib.oracle_num_threads.restype = ctypes.c_int
        lib.oracle_set_threads.argtypes = [ctypes.c_int]
        vp = ctypes.c_void_p
        lib.oracle_generate_words.argtypes = [vp, i64, i64, ctypes.c_uint64, vp, vp, vp,
                                              ctypes.c_uint64, ctypes.c_uint64, vp, i64]
        _lib = lib
    return _lib


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def c_column_sums(words: np.ndarray) -> np.ndarray:
    words = np.ascontiguousarray(words, dtype=np.uint64)
    m, nw = words.shape
    v = np.zeros(m, dtype=np.uint64)
    c_lib().oracle_column_sums(_ptr(words, ctypes.c_uint64), m, nw, _ptr(v, ctypes.c_uint64))
    return v


def c_gram_ones(words: np.ndarray) -> np.ndarray:
    words = np.ascontiguousarray(words, dtype=np.uint64)
    m, nw = words.shape
    out = np.zeros((m, m), dtype=np.int64)
    c_lib().oracle_gram_ones(_ptr(words, ctypes.c_uint64), m, nw, _ptr(out, ctypes.c_int64))
    return out


def c_mi_all_pairs(words: np.ndarray, n_rows: int, mode="exact", epsilon=1e-12,
                   include_diagonal=True, threads: int = 0) -> np.ndarray:
    """Fused C restatement of engine.mi_all_pairs (dense backend), OpenMP-parallel."""
    words = np.ascontiguousarray(words, dtype=np.uint64)
    m, nw = words.shape
    out = np.empty((m, m), dtype=np.float64)
    lib = c_lib()
    if threads:
        lib.oracle_set_threads(int(threads))
    rc = lib.oracle_mi_all_pairs(_ptr(words, ctypes.c_uint64), m, nw, int(n_rows),
                                 MODES.index(mode), float(epsilon), int(bool(include_diagonal)),
                                 _ptr(out, ctypes.c_double))
    if rc != 0:
        raise OracleError(f"oracle_mi_all_pairs failed rc={rc}")
    return out


def c_generate_config_words(recipe: dict, cols=None) -> np.ndarray:
    """Packed words of a config recipe (only `cols` if given), by the C generator."""
    n, m, seed = recipe["n"], recipe["m"], recipe["seed"]
    dens = np.broadcast_to(np.asarray(recipe["density"], dtype=np.float64), (m,))
    thr = np.zeros(m, dtype=np.uint64)
    kind = np.zeros(m, dtype=np.uint8)
    src = np.zeros(m, dtype=np.int32)
    for c in range(m):
        t = threshold(float(dens[c]))
        if t <= 0:
            kind[c] = 1
        elif t >= 1 << 64:
            kind[c] = 2
        else:
            thr[c] = t
    for c in recipe["zero_cols"]:
        kind[c] = 1
    for c in recipe["one_cols"]:
        kind[c] = 2
    for s, t in recipe["pairs"]:
        kind[t] = 3
        src[t] = s
    ft = min(threshold(recipe["flip_density"]), (1 << 64) - 1) if recipe["pairs"] else 0
    sel = None if cols is None else np.ascontiguousarray(np.asarray(cols, dtype=np.int64))
    k = m if sel is None else len(sel)
    words = np.zeros((k, n_words(n)), dtype=np.uint64)
    c_lib().oracle_generate_words(words.ctypes.data, n, m, seed & ((1 << 64) - 1), thr.ctypes.data,
                                  kind.ctypes.data, src.ctypes.data, ft,
                                  (seed ^ FLIP_SEED_XOR) & ((1 << 64) - 1),
                                  None if sel is None else sel.ctypes.data, k)
    return words


def c_num_threads() -> int:
    return int(c_lib().oracle_num_threads())


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


if os.environ.get("MI_ORACLE_IMPORT_GUARD") == "product":  # pragma: no cover
    raise ImportError("oracle imported from a product path")
