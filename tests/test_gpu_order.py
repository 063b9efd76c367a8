"""GPU parity of the column-sum order (mi_column_order, mi_unpack_colsum_ordered,
mi_unpermute): the same matrix as the natural order -- counts bit-exact, MI
within the contract of the oracle -- plus the pieces on their own: the order
is the stable sort of the column sums, and mi_unpermute equals torch indexing
at ragged sizes, pitches, both element sizes and multi-chunk rows.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import rand_bits
from oracle import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def spread_words(n, m, seed, lo=0.0, hi=1.0):
    rng = np.random.default_rng(seed)
    p = rng.uniform(lo, hi, m)
    bits = (rng.random((n, m)) < p[None, :]).astype(np.uint8)
    if m >= 4:
        bits[:, 0] = 0
        bits[:, m - 1] = 1
    return O.pack_bits(bits)


def test_column_order_is_stable_sort(engine):
    from paper_2411_19702_b200 import _native as nat

    for n, m, seed in ((1, 1, 0), (70, 5, 1), (3000, 1025, 2), (999, 4096, 3)):
        words = spread_words(n, m, seed)
        wd = engine.upload(words)
        spread = torch.empty((2,), dtype=torch.int32, device=engine.device)
        perm, inv = engine.column_order(wd, n, m, spread)
        v = O.column_sums(words).astype(np.int64)
        want = np.argsort(v, kind="stable")
        assert np.array_equal(perm.cpu().numpy(), want)
        assert np.array_equal(inv.cpu().numpy()[want], np.arange(m))
        assert tuple(spread.cpu().tolist()) == (int(v.min()), int(v.max()))
    with pytest.raises(Exception):
        nat.check(nat.lib().mi_column_order(None, 10, 10, None, None, None, None), "mi_column_order")


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.int32])
def test_unpermute_matches_indexing(engine, dtype):
    from paper_2411_19702_b200 import _native as nat

    dev = engine.device
    g = torch.Generator(device="cpu").manual_seed(5)
    for m, pad_in, pad_out in ((1, 0, 0), (2, 1, 0), (3, 0, 5), (255, 0, 0), (257, 3, 1), (777, 0, 2), (4100, 0, 0),
                               (8, 0, 0), (148, 4, 0), (1000, 0, 4), (1002, 2, 2), (10_000, 0, 0), (150, 0, 0)):
        src = torch.randn((m, m + pad_in), generator=g).to(dtype if dtype != torch.int32 else torch.float64)
        if dtype == torch.int32:
            src = (src * 1e6).to(torch.int32)
        src = src.to(dev)
        inv = torch.randperm(m, generator=g).to(torch.int32).to(dev)
        out = torch.full((m, m + pad_out), -7, dtype=dtype, device=dev)
        nat.check(nat.lib().mi_unpermute(src.data_ptr(), src.stride(0), out.data_ptr(), out.stride(0), m,
                                         src.element_size(), inv.data_ptr(),
                                         torch.cuda.current_stream(dev).cuda_stream), "mi_unpermute")
        il = inv.long()
        want = src[:, :m].index_select(0, il).index_select(1, il)
        assert torch.equal(out[:, :m], want), (m, pad_in, pad_out)
        if pad_out:
            assert bool((out[:, m:] == -7).all()), "wrote past n_cols"


def test_unpermute_multi_chunk_rows(engine):
    """Rows larger than a CTA's shared memory are staged in several chunks."""
    from paper_2411_19702_b200 import _native as nat

    dev = engine.device
    nat.set_tuning(unperm_ctas=4)  # ~56 KB per CTA: a 9000-element float64 row takes 2 chunks
    try:
        m = 9000
        g = torch.Generator(device="cpu").manual_seed(9)
        src = torch.randn((m, m), generator=g, dtype=torch.float64).to(dev)
        inv = torch.randperm(m, generator=g).to(torch.int32).to(dev)
        out = torch.empty_like(src)
        nat.check(nat.lib().mi_unpermute(src.data_ptr(), m, out.data_ptr(), m, m, 8, inv.data_ptr(),
                                         torch.cuda.current_stream(dev).cuda_stream), "mi_unpermute")
        il = inv.long()
        assert torch.equal(out, src.index_select(0, il).index_select(1, il))
    finally:
        nat.set_tuning(unperm_ctas=0)


def test_unpermute_rejects_bad_arguments(engine):
    from paper_2411_19702_b200 import _native as nat
    from paper_2411_19702_b200.errors import DimensionError, DomainError

    t = torch.zeros((8, 8), dtype=torch.float64, device=engine.device)
    inv = torch.arange(8, dtype=torch.int32, device=engine.device)
    L = nat.lib()
    with pytest.raises(DomainError):
        nat.check(L.mi_unpermute(t.data_ptr(), 8, t.data_ptr(), 8, 8, 8, inv.data_ptr(), None), "overlap")
    with pytest.raises(DomainError):
        nat.check(L.mi_unpermute(t.data_ptr(), 8, t.data_ptr(), 8, 8, 2, inv.data_ptr(), None), "esz")
    with pytest.raises(DimensionError):
        nat.check(L.mi_unpermute(t.data_ptr(), 4, t.data_ptr(), 8, 8, 8, inv.data_ptr(), None), "ld")


@pytest.mark.parametrize("n,m,seed", [(3000, 700, 11), (257, 513, 12), (4097, 1100, 13), (64, 300, 14)])
def test_colsum_order_matches_oracle(engine, n, m, seed):
    words = spread_words(n, m, seed)
    wd = engine.upload(words)
    ref = O.c_mi_all_pairs(words, n)
    for dtype, tol in ((torch.float64, 1e-12), (torch.float32, 1e-6)):
        got = engine.all_pairs_device(wd, n, m, None, dtype, order="colsum").double().cpu().numpy()
        assert float(np.max(np.abs(got - ref))) < tol
        assert np.array_equal(got, got.T)
    prep = engine.prepare(wd, n, m, order="colsum")
    g = engine.compute(prep, None, torch.int32).cpu().numpy().astype(np.int64)
    assert np.array_equal(g, O.c_gram_ones(words)), "counts differ under the column-sum order"
    nodiag = engine.compute(prep, _cfg(diag=False), torch.float64).cpu().numpy()
    assert np.all(np.diagonal(nodiag) == 0.0)
    r2 = ref.copy()
    np.fill_diagonal(r2, 0.0)
    assert float(np.max(np.abs(nodiag - r2))) < 1e-12
    eps = engine.compute(prep, _cfg(mode="epsilon"), torch.float64).cpu().numpy()
    ref_eps = O.c_mi_all_pairs(words, n, mode="epsilon", epsilon=1e-12)
    assert float(np.max(np.abs(eps - ref_eps))) < 1e-12


def _cfg(mode="exact", eps=1e-12, diag=True):
    from paper_2411_19702_b200 import EngineConfig

    return EngineConfig(mode=mode, epsilon=eps, include_diagonal=diag)


def test_colsum_order_golden_values(engine):
    """Exact golden values survive the reordering (balanced copies -> 1.0)."""
    rng = np.random.default_rng(3)
    n, m = 4000, 600
    bits = rand_bits(rng, n, m, 0.3)
    bits[:, 10] = (np.arange(n) % 2).astype(np.uint8)
    bits[:, 500] = bits[:, 10]
    bits[:, 20] = 0
    bits[:, 30] = 1
    bits[:, 40:140] = (rng.random((n, 100)) < 0.9).astype(np.uint8)
    words = O.pack_bits(bits)
    got = engine.all_pairs_device(engine.upload(words), n, m, order="colsum").cpu().numpy()
    assert got[10, 500] == 1.0 and got[500, 10] == 1.0
    assert np.all(got[20] == 0.0) and np.all(got[:, 30] == 0.0)
    assert float(np.max(np.abs(got - O.c_mi_all_pairs(words, n)))) < 1e-12


def test_auto_rule(engine):
    from paper_2411_19702_b200.errors import DomainError

    rng = np.random.default_rng(1)
    clustered = O.pack_bits(rand_bits(rng, 20000, 600, 0.5))          # spread ~ 600 < table_thr
    spread = spread_words(20000, 600, 2)                               # spread ~ 20000
    from paper_2411_19702_b200 import engine as E

    old = E.AUTO_ORDER_MIN_COLS
    E.AUTO_ORDER_MIN_COLS = 512
    try:
        assert engine.choose_order(engine.upload(clustered), 20000, 600) == "natural"
        assert engine.choose_order(engine.upload(spread), 20000, 600) == "colsum"
        assert engine.choose_order(engine.upload(spread), 20000, 600, world=2) == "natural"
    finally:
        E.AUTO_ORDER_MIN_COLS = old
    assert engine.choose_order(engine.upload(spread), 20000, 600) == "natural"  # narrower than the default bound
    assert engine.choose_order(engine.upload(spread_words(20000, 200, 3)), 20000, 200) == "natural"  # one tile
    wd = engine.upload(spread)
    with pytest.raises(DomainError):
        engine.prepare(wd, 20000, 600, rank=0, world=2, order="colsum")
    with pytest.raises(DomainError):
        engine.prepare(wd, 20000, 600, order="sorted")
    prep = engine.prepare(wd, 20000, 600, order="colsum")
    with pytest.raises(DomainError):
        engine.compute(prep, None, torch.float64, packed=True)


@pytest.mark.parametrize("cfg", [2, 4])
def test_colsum_order_full_config(engine, cfg):
    """Configs 2 and 4 at full size: the column-sum order gives the natural
    order's matrix (counts-exact table path vs FP64 path: within 1e-12 for
    float64, 1e-6 for float32) and matches the oracle on a column subset."""
    from paper_2411_19702_b200 import datagen

    rec = datagen.config_recipe(cfg)
    n, m = rec["n"], rec["m"]
    dt = torch.float64 if datagen.CONFIGS[cfg]["out"] == "float64" else torch.float32
    words = datagen.generate_words_device(rec, engine.device)
    assert engine.choose_order(words, n, m) == ("colsum" if m >= 16384 else "natural")
    a = engine.all_pairs_device(words, n, m, None, dt, order="natural")
    b = engine.all_pairs_device(words, n, m, None, dt, order="colsum")
    tol = 1e-12 if dt == torch.float64 else 1e-6
    step = 4096
    for r0 in range(0, m, step):
        assert (a[r0:r0 + step].double() - b[r0:r0 + step].double()).abs().max().item() < tol
    del a
    assert torch.equal(b, b.T)
    rng = np.random.default_rng(cfg)
    S = np.unique(np.concatenate([rng.choice(m, 300, replace=False), [0, 255, 256, m - 1],
                                  np.array(rec["pairs"][:20], dtype=np.int64).ravel()]))
    idx = torch.from_numpy(S).to(engine.device)
    wS = words.index_select(0, idx).cpu().numpy().view(np.uint64)
    got = b.index_select(0, idx).index_select(1, idx).double().cpu().numpy()
    assert float(np.max(np.abs(got - O.c_mi_all_pairs(wS, n)))) < tol
    del b, words
    torch.cuda.empty_cache()


def test_slot_order_output(engine):
    """compute_slot_order: S[a, b] = MI(perm[a], perm[b]) without the unpermute."""
    from paper_2411_19702_b200.errors import DomainError

    n, m = 3000, 900
    words = spread_words(n, m, 21)
    wd = engine.upload(words)
    full = engine.all_pairs_device(wd, n, m, order="colsum").cpu().numpy()
    prep = engine.prepare(wd, n, m, order="colsum")
    S, perm = engine.compute_slot_order(prep)
    S, perm = S.cpu().numpy(), perm.cpu().numpy().astype(np.int64)
    assert np.array_equal(S, full[np.ix_(perm, perm)])
    with pytest.raises(DomainError):
        engine.compute_slot_order(engine.prepare(wd, n, m))
