"""The operand-format boundary: e2m1 operands with fp32 accumulators hold
exact counts only below 2^24 rows, so N = 2^24 - 1 is the largest e2m1 case
(counts up to 2^24 - 1, all-ones columns hit it) and N = 2^24 + 77 runs the
int8 path (and the FP64 epilogue: the fixed-point table also stops at 2^24).
Counts bit-exact and MI within 1e-12 against the C oracle on all columns.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _words(n: int, m: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    nw = (n + 63) // 64
    w = rng.integers(0, 2**63, size=(m, nw), dtype=np.int64).view(np.uint64)
    w[:, :] ^= rng.integers(0, 2, size=(m, nw), dtype=np.uint64) << np.uint64(63)
    w[0, :] = np.uint64(0xFFFFFFFFFFFFFFFF)   # all ones: the largest count, N
    w[1, :] = np.uint64(0)                    # all zeros
    w[2, :] = w[0, :]                         # identical to column 0
    w[3, :] = w[4, :]                         # identical random columns
    sparse = rng.random((m - 40, nw)) < 0.02  # a few very sparse columns
    w[40:, :] &= np.where(sparse, w[40:, :], np.uint64(0))
    tail = n % 64
    if tail:
        w[:, -1] &= np.uint64((1 << tail) - 1)
    return w


@pytest.mark.parametrize("n,fmt", [((1 << 24) - 1, "e2m1"), ((1 << 24) + 77, "int8")])
def test_operand_format_boundary(engine, n, fmt):
    from paper_2411_19702_b200 import _native as nat

    m = 72
    words = _words(n, m, seed=n % 1000)
    ld = int(nat.lib().mi_kmajor_ld(n))
    if fmt == "e2m1":
        assert ld == ((n + 255) // 256) * 128
    else:
        assert ld == ((n + 127) // 128) * 128
    dev = engine.upload(words)
    g, v = engine.gram_counts(dev, n, m)
    g = g.cpu().numpy().astype(np.int64)
    assert np.array_equal(v.cpu().numpy().astype(np.uint64), O.c_column_sums(words))
    assert g[0, 0] == n and g[0, 2] == n and g[1, 1] == 0
    assert np.array_equal(g, O.c_gram_ones(words))
    mi = engine.all_pairs_device(dev, n, m).cpu().numpy()
    ref = O.c_mi_all_pairs(words, n)
    assert np.array_equal(mi, mi.T)
    assert float(np.max(np.abs(mi - ref))) < 1e-12
    del dev
    torch.cuda.empty_cache()


def test_int8_path_multi_tile_above_2e24(engine):
    """N = 2^24 + 77 (int8 operands, kind::i8, s32 accumulators, FP64
    epilogue) at m = 700: three tile rows, ragged last tile, the tail split of
    the last round.  Counts bit-exact and MI within 1e-12 against the C
    oracle on a column subset that spans every tile boundary (MI(i, j)
    depends only on columns i and j)."""
    n, m = (1 << 24) + 77, 700
    words = _words(n, m, seed=7)
    dev = engine.upload(words)
    g, v = engine.gram_counts(dev, n, m)
    assert np.array_equal(v.cpu().numpy().astype(np.uint64), O.c_column_sums(words))
    mi = engine.all_pairs_device(dev, n, m).cpu().numpy()
    assert np.array_equal(mi, mi.T)
    cols = np.array(sorted({0, 1, 2, 3, 4, 5, 41, 127, 128, 255, 256, 257, 383, 384, 511, 512, 513, 600, 698, 699}))
    sub = np.ascontiguousarray(words[cols])
    gs = g.cpu().numpy().astype(np.int64)[np.ix_(cols, cols)]
    assert np.array_equal(gs, O.c_gram_ones(sub))
    ref = O.c_mi_all_pairs(sub, n)
    assert float(np.max(np.abs(mi[np.ix_(cols, cols)] - ref))) < 1e-12
    del dev, g
    torch.cuda.empty_cache()
