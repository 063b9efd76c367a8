"""The word-operand path (mi_colstat_words + mi_gram_mi_words): the fused
kernel's producer warps expand the packed words into the swizzled stages
themselves, so X never exists in HBM (tall-N / narrow-m shapes).

Its operands hold the same 0/1 bits in a different K order (any bijection of
rows onto K slots shared by both operands leaves every dot product unchanged),
so counts are exact integers either way and every output -- counts, float64,
float32, epsilon mode, packed, tile-major, the host entry points -- must be
bit-identical to the unpack + TMA path, and match the oracle
(/root/reference/pkg/src/mimatrix/_kernels.py:36-61 reads the same words).
"""

from __future__ import annotations

import contextlib

import numpy as np
import pytest

from conftest import rand_bits
from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@contextlib.contextmanager
def knobs(**kw):
    from paper_2411_19702_b200 import _native as nat

    old = {k: nat.get_tuning(k) for k in kw}
    try:
        nat.set_tuning(**kw)
        yield
    finally:
        nat.set_tuning(**old)


def both_paths(engine, words, n, fn):
    """fn(words_dev) under xp = 1 (word operand) and xp = 0 (unpack + TMA)."""
    m = words.shape[0]
    w = engine.upload(words)
    with knobs(xp=1):
        # (odd word counts per column run on a padded copy: the TMA row pitch
        # must be a multiple of 16 bytes)
        assert engine.words_operand(n, m)
        a = fn(w)
    with knobs(xp=0):
        assert not engine.words_operand(n, m)
        b = fn(w)
    return a, b


def cfg_of(mode="exact", eps=1e-12, diag=True):
    from paper_2411_19702_b200 import EngineConfig

    return EngineConfig(mode=mode, epsilon=eps, include_diagonal=diag)


SHAPES = [
    (1, 1, 1.0), (300, 5, 0.5), (1000, 257, 0.3), (4099, 511, 0.5), (4200, 511, 0.5), (20_000, 700, 0.1),
    (129, 1, 0.5), (1_000_000, 100, 0.5),
    (70_001, 513, 0.45), (250_000, 256, 0.5), (600_000, 300, 0.02), (64 * 4 * 77 + 64, 600, 0.7),
    # even word counts (no padded copy): tiny m, m below one
    # 128-row half, ragged K tails, tall N
    (128, 1, 0.5), (1024, 5, 0.7), (8192, 100, 0.2), (6400, 130, 0.5), (65_536 + 128, 255, 0.4),
    (1_000_064, 64, 0.5), (300_032, 1023, 0.05),
]


@pytest.mark.parametrize("n,m,d", SHAPES, ids=lambda v: str(v))
def test_counts_and_mi_bit_identical_to_unpack_path(engine, n, m, d):
    rng = np.random.default_rng(n * 7 + m)
    words = O.pack_bits(rand_bits(rng, n, m, d))

    def run(w):
        prep = engine.prepare(w, n, m)
        g = engine.compute(prep, None, torch.int32).cpu().numpy()
        f64 = engine.compute(prep, None, torch.float64).cpu().numpy()
        f32 = engine.compute(prep, None, torch.float32).cpu().numpy()
        eps = engine.compute(prep, cfg_of("epsilon", 1e-9, False), torch.float64).cpu().numpy()
        return g, f64, f32, eps, prep.colsum[:m].cpu().numpy()

    a, b = both_paths(engine, words, n, run)
    for x, y, what in zip(a, b, ("counts", "f64", "f32", "epsilon", "colsum")):
        assert np.array_equal(x, y), what
    if n * m * m <= 4e11:
        assert np.array_equal(a[0].astype(np.int64), O.c_gram_ones(words))
        ref = O.c_mi_all_pairs(words, n)
        assert float(np.max(np.abs(a[1] - ref))) < 1e-12
        assert float(np.max(np.abs(a[2] - ref))) < 1e-6


@pytest.mark.parametrize("tail", [0, 2, 3])
@pytest.mark.parametrize("n,m", [(2_000_000, 512), (40_000, 1800), (3000, 3000)])
def test_tail_schedules(engine, tail, n, m):
    """Narrow m is all tail: 3 tiles at m = 512 run as K ranges over the SM
    pairs; column slices and the unsplit schedule agree bit for bit."""
    rng = np.random.default_rng(tail + n)
    words = O.pack_bits(rand_bits(rng, n, m, 0.35))
    with knobs(tail=tail):
        a, b = both_paths(engine, words, n, lambda w: engine.all_pairs_device(w, n, m, None, torch.float64).cpu().numpy())
    assert np.array_equal(a, b)
    assert np.array_equal(a, a.T)


def test_output_forms_and_tile_subsets(engine):
    from paper_2411_19702_b200.engine import unpack_upper

    n, m = 90_112, 1000
    rng = np.random.default_rng(17)
    words = O.pack_bits(rand_bits(rng, n, m, 0.25))

    def run(w):
        prep = engine.prepare(w, n, m)
        full = engine.compute(prep, None, torch.float64).cpu().numpy()
        packed = engine.compute(prep, None, torch.float64, packed=True).cpu().numpy()
        tl = engine.tiles(m, 1, 3)
        # (cells past m in the last block are never written: start from zeros)
        shard = torch.zeros((int(tl.shape[0]), 256, 256), dtype=torch.float32, device=engine.device)
        shard = engine.compute(prep, None, torch.float32, tiles=tl, tile_major=True, out=shard).cpu().numpy()
        return full, packed, shard

    a, b = both_paths(engine, words, n, run)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert np.array_equal(unpack_upper(a[1], m), a[0])


def test_host_entry_points(engine):
    """mi_all_pairs_host (staged ingest and row-band egress), the packed host
    call and mi_gram_ones_host through the word-operand path."""
    from paper_2411_19702_b200 import BinaryMatrix, gram_ones, mi_all_pairs, mi_all_pairs_c_abi

    n, m = 300_000, 700
    rng = np.random.default_rng(23)
    words = O.pack_bits(rand_bits(rng, n, m, 0.4))
    mat = BinaryMatrix(n, m, words)
    res = {}
    for xp in (1, 0):
        with knobs(xp=xp):
            r = [mi_all_pairs(mat).values, mi_all_pairs_c_abi(mat, out_dtype=np.float32), gram_ones(mat)]
            with knobs(ingest=0):
                r.append(mi_all_pairs(mat).values)
            r.append(engine.all_pairs_host(words, n, m, packed=True))
            res[xp] = r
    for x, y in zip(res[1], res[0]):
        assert np.array_equal(x, y)
    assert np.array_equal(res[1][0], res[1][3])
    assert np.array_equal(res[1][2], O.c_gram_ones(words))


def test_staged_prepare_ranges(engine):
    """prepare_begin / prepare_range (the staged broadcast's per-group
    statistics) feed the word-operand GEMM too."""
    n, m = 50_000, 1500
    rng = np.random.default_rng(31)
    words = O.pack_bits(rand_bits(rng, n, m, 0.5))

    def run(w):
        prep = engine.prepare_begin(n, m)
        cuts = [0, 512, 1024, prep.m_pad]
        for c0, c1 in zip(cuts, cuts[1:]):
            engine.prepare_range(prep, w, c0, c1)
        return engine.compute(prep, None, torch.float64).cpu().numpy()

    a, b = both_paths(engine, words, n, run)
    assert np.array_equal(a, b)


def test_default_rule_picks_words_for_narrow_m(engine):
    with knobs(xp=-1):
        assert engine.words_operand(8_000_000, 512)
        assert engine.words_operand(102_400, 2048)
        assert engine.words_operand(8_000_064, 512)       # odd word count: padded copy, still ahead
        assert not engine.words_operand(100_000, 2048)    # odd word count, wider: the unpack path
        assert not engine.words_operand(100_000, 10_000)
        assert not engine.words_operand((1 << 24) + 1, 256)  # int8 operands: no word build


def test_layout_knob_change_between_prepare_and_compute_is_rejected(engine):
    """X's format is fixed by the fp4 / cta_group knobs at prepare time; a
    compute() under other knobs would read it wrongly, so it raises."""
    from paper_2411_19702_b200 import DomainError

    n, m = 5000, 5000  # the unpack path (m_pad > xp_cols)
    rng = np.random.default_rng(3)
    w = engine.upload(O.pack_bits(rand_bits(rng, n, m, 0.5)))
    prep = engine.prepare(w, n, m)
    with knobs(fp4=0):
        with pytest.raises(DomainError):
            engine.compute(prep, None, torch.float64)
    engine.compute(prep, None, torch.float64)  # unchanged knobs: fine


@pytest.mark.parametrize("n,m", [(300_000, 512), (2_000_000, 1000), (70_016, 700), (1_000_000, 256)])
def test_statistics_inside_the_fused_launch(engine, n, m):
    """xp_stats = 1: for the full tile list of a narrow matrix the column
    statistics are computed inside the fused launch (the expanders count the
    diagonal units' columns, the epilogue warps build the statistics behind
    grid-wide barriers); every output equals the separate counting pass's."""
    rng = np.random.default_rng(n + 3 * m)
    dens = rng.uniform(0.02, 0.98, size=m)
    bits = (rng.random((n, m)) < dens[None, :]).astype(np.uint8)
    bits[:, 0] = 0
    bits[:, 1] = 1
    words = O.pack_bits(bits)
    w = engine.upload(words)
    cases = [(None, torch.float64), (None, torch.float32), (None, torch.int32),
             (cfg_of("epsilon", 1e-9, False), torch.float64)]
    res = {}
    for xs in (1, 0):
        with knobs(xp=1, xp_stats=xs):
            outs = []
            for cfg, dt in cases:
                prep = engine.prepare(w, n, m)  # fresh: the first compute computes the statistics
                outs.append(engine.compute(prep, cfg, dt).cpu().numpy())
                outs.append(prep.colsum[:m].cpu().numpy())
            res[xs] = outs
    for a, b in zip(res[1], res[0]):
        assert np.array_equal(a, b)
    assert np.array_equal(res[1][1].astype(np.uint64), bits.sum(axis=0).astype(np.uint64))


def test_host_paths_with_fused_statistics(engine):
    from paper_2411_19702_b200 import BinaryMatrix, gram_ones, mi_all_pairs

    n, m = 400_000, 600
    rng = np.random.default_rng(77)
    words = O.pack_bits(rand_bits(rng, n, m, 0.35))
    mat = BinaryMatrix(n, m, words)
    res = {}
    for xs in (1, 0):
        with knobs(xp=1, xp_stats=xs, ingest=0):
            res[xs] = [mi_all_pairs(mat).values, gram_ones(mat)]
    for a, b in zip(res[1], res[0]):
        assert np.array_equal(a, b)
