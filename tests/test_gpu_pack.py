"""Device packing (mi_pack_bits, MIEngine.pack_bits): the reference's
from_bits / from_rows layout bit for bit, at ragged shapes and pitches, with
from_rows's rejection of non-binary values (binmat.py:34-46,136-172)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("n,m", [(1, 1), (63, 5), (64, 128), (65, 129), (255, 300), (256, 127), (1000, 700),
                                 (4097, 1300), (20_000, 257)])
def test_pack_matches_reference_layout(engine, n, m):
    rng = np.random.default_rng(n + 31 * m)
    bits = (rng.random((n, m)) < rng.uniform(0, 1)).astype(np.uint8)
    words = engine.pack_bits(torch.from_numpy(bits).to(engine.device)).cpu().numpy().view(np.uint64)
    assert np.array_equal(words, O.pack_bits(bits))
    # a pitched view (row stride > m) and bool input give the same words
    wide = np.zeros((n, m + 13), dtype=np.uint8)
    wide[:, :m] = bits
    view = torch.from_numpy(wide).to(engine.device)[:, :m]
    assert np.array_equal(engine.pack_bits(view).cpu().numpy().view(np.uint64), words)
    as_bool = torch.from_numpy(bits.astype(bool)).to(engine.device)
    assert np.array_equal(engine.pack_bits(as_bool).cpu().numpy().view(np.uint64), words)


def test_pack_then_mi_end_to_end(engine):
    rng = np.random.default_rng(5)
    n, m = 3000, 600
    bits = (rng.random((n, m)) < 0.3).astype(np.uint8)
    w = engine.pack_bits(torch.from_numpy(bits).to(engine.device))
    mi = engine.all_pairs_device(w, n, m).cpu().numpy()
    assert float(np.max(np.abs(mi - O.c_mi_all_pairs(O.pack_bits(bits), n)))) < 1e-12


def test_pack_rejects_non_binary(engine):
    from paper_2411_19702_b200.errors import DimensionError, DomainError

    bits = np.zeros((300, 200), dtype=np.uint8)
    bits[123, 45] = 2
    with pytest.raises(DomainError):
        engine.pack_bits(torch.from_numpy(bits).to(engine.device))
    with pytest.raises(DimensionError):
        engine.pack_bits(torch.zeros((4, 4), dtype=torch.int32, device=engine.device))


def test_pack_transposed_and_single_row_views(engine):
    rng = np.random.default_rng(12)
    bits = (rng.random((300, 1)) < 0.5).astype(np.uint8)
    for arr in (bits, bits.T, np.asfortranarray((rng.random((50, 70)) < 0.5).astype(np.uint8))):
        t = torch.from_numpy(np.asarray(arr)).to(engine.device)
        if arr.shape[1] > 1:
            t = torch.from_numpy(np.ascontiguousarray(arr).T.copy()).to(engine.device).T  # column-major view
        w = engine.pack_bits(t).cpu().numpy().view(np.uint64)
        assert np.array_equal(w, O.pack_bits(np.ascontiguousarray(t.cpu().numpy())))


def test_engine_from_bits_host(engine):
    from paper_2411_19702_b200.binmat import from_bits
    from paper_2411_19702_b200.errors import DomainError

    rng = np.random.default_rng(8)
    bits = (rng.random((5000, 777)) < 0.4).astype(np.uint8)
    got = engine.from_bits(bits)
    want = from_bits(bits)
    assert got.n_rows == want.n_rows and got.n_cols == want.n_cols
    assert np.array_equal(got.words, want.words)
    assert np.array_equal(engine.from_bits(bits.astype(np.int64)).words, want.words)
    assert np.array_equal(engine.from_bits(bits.astype(bool)).words, want.words)
    bad = bits.astype(np.int64)
    bad[3, 3] = 5
    with pytest.raises(DomainError):
        engine.from_bits(bad)
    bad8 = bits.copy()
    bad8[10, 20] = 2
    with pytest.raises(DomainError):
        engine.from_bits(bad8)


class _Sparse:
    """The reference's SparseBinaryMatrix shape (binmat.py:100-133): per-column
    sorted row-index lists."""

    def __init__(self, n, m, cols):
        self.n_rows, self.n_cols, self.col_indices = n, m, tuple(cols)


def _sparse_of(bits):
    return _Sparse(bits.shape[0], bits.shape[1], [np.flatnonzero(bits[:, j]).astype(np.int64)
                                                  for j in range(bits.shape[1])])


@pytest.mark.parametrize("n,m,d", [(1, 1, 1.0), (63, 3, 0.5), (65, 40, 0.3), (1000, 257, 0.01), (20_000, 600, 0.002),
                                   (4096, 33, 0.0), (777, 129, 1.0)])
def test_pack_sparse_matches_dense(engine, n, m, d):
    """binmat.to_dense on the device: the index lists give the same words as
    packing the dense matrix, and the drop-in / gram_ones / column_sums on
    sparse input equal the dense results."""
    from paper_2411_19702_b200 import BinaryMatrix, column_sums, gram_ones, mi_all_pairs

    rng = np.random.default_rng(n * 31 + m)
    bits = (rng.random((n, m)) < d).astype(np.uint8)
    sp = _sparse_of(bits)
    words = engine.from_sparse(sp).cpu().numpy().view(np.uint64)
    assert np.array_equal(words, O.pack_bits(bits))
    dense = BinaryMatrix(n, m, O.pack_bits(bits))
    assert np.array_equal(mi_all_pairs(sp, backend="sparse").values, mi_all_pairs(dense).values)
    assert np.array_equal(gram_ones(sp), gram_ones(dense))
    assert np.array_equal(column_sums(sp), column_sums(dense))


def test_pack_sparse_rejects_out_of_range(engine):
    from paper_2411_19702_b200 import DomainError

    with pytest.raises(DomainError):
        engine.from_sparse(_Sparse(10, 2, [np.array([0, 3]), np.array([10])]))
