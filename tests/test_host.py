"""Host-side logic and the C-ABI boundary, without a GPU.

No compute calls: only loading the library, checking its exports, the pure
host helpers (layout, tile lists) and argument validation that fails before
any device work.
"""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from conftest import rand_bits
from oracle import oracle as O
from paper_2411_19702_b200 import (
    BACKENDS,
    BinaryMatrix,
    DimensionError,
    DomainError,
    EngineConfig,
    NativeError,
    from_bits,
    from_rows,
    mi_all_pairs,
)
from paper_2411_19702_b200 import _native as nat
from paper_2411_19702_b200 import datagen, dispatch


# ------------------------------------------------------------------ C ABI
def test_library_exports_every_header_function():
    lib = nat.lib()
    declared = nat.header_functions()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/mimatrix_b200.h but not exported"
    assert set(declared) == set(nat.SIGNATURES), "ctypes signatures out of sync with the header"
    assert lib.mi_b200_abi_version() == 1


def test_layout_helpers():
    lib = nat.lib()
    old = nat.get_tuning("fp4")
    try:
        nat.set_tuning(fp4=0)  # int8 operand: one byte per row, rows padded to 128
        assert lib.mi_kmajor_ld(1) == 128 and lib.mi_kmajor_ld(128) == 128 and lib.mi_kmajor_ld(129) == 256
        nat.set_tuning(fp4=1)  # e2m1 operand: two rows per byte, rows padded to 256
        assert lib.mi_kmajor_ld(1) == 128 and lib.mi_kmajor_ld(256) == 128 and lib.mi_kmajor_ld(257) == 256
        assert lib.mi_kmajor_ld((1 << 24) + 1) == (1 << 24) + 128  # fp32-exactness limit: back to int8
    finally:
        nat.set_tuning(fp4=old)
    assert lib.mi_kmajor_rows(1) == 256 and lib.mi_kmajor_rows(257) == 512
    assert lib.mi_tile_size() in (128, 256)
    T = -(-10000 // lib.mi_tile_size())
    assert lib.mi_num_tiles(10000) == T * (T + 1) // 2
    assert lib.mi_colstat_bytes(1000, 300) == 512 * 112 + 1001 * 8 + 4 * 8 + 1024 * 12
    assert lib.mi_colstat_bytes(1 << 25, 300) == 512 * 112


@pytest.mark.parametrize("m", [1, 255, 256, 257, 1000, 10000, 50000])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_tile_partition_covers_triangle_once(m, world):
    lib = nat.lib()
    T = -(-m // lib.mi_tile_size())
    seen = {}
    counts = []
    for r in range(world):
        tl = nat.tile_list(m, r, world)
        counts.append(len(tl))
        for I, J in tl.tolist():
            assert 0 <= I <= J < T
            assert (I, J) not in seen, "tile dealt twice"
            seen[(I, J)] = r
    assert len(seen) == T * (T + 1) // 2
    if world == 8 and T >= 8:  # column-group pairs, the diagonal ranks' surplus handed on
        assert max(counts) <= -(-len(seen) // 8), "a share above ceil(tiles / 8)"
        assert max(counts) - min(counts) <= T // 4 + 2, "unbalanced shares"
    else:
        assert max(counts) - min(counts) <= 1, "unbalanced shares"


@pytest.mark.parametrize("m", [2048, 10000, 50000])
def test_eight_rank_column_groups_halve_the_footprint(m):
    lib = nat.lib()
    t = lib.mi_tile_size()
    T = -(-m // t)
    for r in range(8):
        mask = nat.rank_blocks(m, r, 8)
        assert mask.shape == (T,)
        used = set(np.flatnonzero(mask).tolist())
        touched = {b for I, J in nat.tile_list(m, r, 8).tolist() for b in (I, J)}
        assert used == touched
        assert len(used) <= T // 2 + 2
    assert nat.rank_blocks(m, 0, 2).sum() == T  # round robin: every block


def test_tile_mask_covers_matrix():
    m = 600
    full = np.zeros((m, m), dtype=int)
    for r in range(3):
        full += dispatch.tile_mask(m, nat.tile_list(m, r, 3))
    assert np.all(full >= 1)
    # an element is written by exactly one rank (tile + mirror of the same tile)
    disjoint = np.zeros((m, m), dtype=int)
    for r in range(3):
        tl = nat.tile_list(m, r, 3)
        t = nat.lib().mi_tile_size()
        for I, J in tl.tolist():
            disjoint[I * t:(I + 1) * t, J * t:(J + 1) * t] += 1
    assert np.all(np.triu(disjoint[:m, :m]) <= 1)


def test_c_abi_rejects_bad_arguments_without_device_work():
    lib = nat.lib()
    assert lib.mi_tile_list(100, 3, 2, 0, None, 0) < 0
    assert lib.mi_tile_list(0, 0, 1, 0, None, 0) < 0
    rc = lib.mi_gram_mi(None, None, 0, 10, 128, 0, 1e-12, 1, 1, None, 10, None, 1, None)
    assert rc == nat.MI_ERR_DIMENSION
    rc = lib.mi_gram_mi(None, None, 10, 10, 128, 7, 1e-12, 1, 1, None, 10, None, 1, None)
    assert rc == nat.MI_ERR_DOMAIN and "mode" in nat.last_error()
    rc = lib.mi_gram_mi(None, None, 10, 10, 128, 1, 0.0, 1, 1, None, 10, None, 1, None)
    assert rc == nat.MI_ERR_DOMAIN
    rc = lib.mi_gram_mi(None, None, 10, 10, 64, 0, 1e-12, 1, 1, None, 10, None, 1, None)
    assert rc == nat.MI_ERR_DIMENSION
    with pytest.raises(DomainError):
        nat.check(nat.MI_ERR_DOMAIN, "x")
    # column ranges must start and end on multiples of 32 (colstat_kernel's warp reductions)
    ld = int(lib.mi_kmajor_ld(1000))
    for c0, c1 in ((0, 40), (16, 64), (64, 32), (0, 544)):
        rc = lib.mi_unpack_colsum_range(None, 1000, 300, None, ld, 1, None, None, c0, c1, None)
        assert rc == nat.MI_ERR_DIMENSION and "multiples of 32" in nat.last_error(), (c0, c1)
    words = np.array([[0b111]], dtype=np.uint64)  # dirty padding for n_rows = 2
    out = np.empty((1, 1))
    rc = lib.mi_all_pairs_host(words.ctypes.data, 2, 1, 0, 1e-12, 1, 1, out.ctypes.data, 0)
    assert rc == nat.MI_ERR_DOMAIN and "padding" in nat.last_error()


def test_words_operand_rule():
    """The word-operand (XP) dispatch rule (capi_common.cu words_operand):
    e2m1 operands only (N < 2^24), m_pad <= xp_cols, a third of that for an
    odd word count per column; xp=0 never, xp=1 always (host logic)."""
    lib = nat.lib()
    old = {k: nat.get_tuning(k) for k in ("xp", "xp_cols")}
    try:
        nat.set_tuning(xp=-1, xp_cols=3072)
        assert lib.mi_words_operand(8_000_000, 512) == 1        # even word count
        assert lib.mi_words_operand(8_000_000, 3072) == 1
        assert lib.mi_words_operand(8_000_000, 3073) == 0       # m_pad 3328 > 3072
        assert lib.mi_words_operand(8_000_064, 512) == 1        # odd word count: m_pad <= 1024
        assert lib.mi_words_operand(8_000_064, 1024) == 1
        assert lib.mi_words_operand(8_000_064, 1025) == 0
        assert lib.mi_words_operand(1 << 24, 512) == 0          # int8 operands beyond 2^24 rows
        assert lib.mi_words_operand(50_000, 50_000) == 0        # config 4: the unpack path
        nat.set_tuning(xp=0)
        assert lib.mi_words_operand(8_000_000, 512) == 0
        nat.set_tuning(xp=1)
        assert lib.mi_words_operand(8_000_000, 50_000) == 1
        assert lib.mi_words_operand(1 << 24, 512) == 0          # never without e2m1 operands
    finally:
        nat.set_tuning(**old)


def test_new_entry_points_reject_bad_arguments_without_device_work():
    """Word-operand, sparse-ingest and multi-device entry points validate
    their arguments before any device call."""
    lib = nat.lib()
    rc = lib.mi_gram_mi_words(None, None, 100, 10, 0, 1e-12, 1, 1, None, 10, None, 1, None)
    assert rc == nat.MI_ERR_DOMAIN and "required" in nat.last_error()
    rc = lib.mi_gram_mi_words_stats(None, None, None, 100, 10, 0, 1e-12, 1, 1, None, 10, None, 1, None)
    assert rc == nat.MI_ERR_DOMAIN
    assert lib.mi_pack_sparse(None, None, 0, 10, None, None, None) == nat.MI_ERR_DIMENSION
    assert lib.mi_pack_sparse(None, None, 10, 10, None, None, None) == nat.MI_ERR_DOMAIN
    words = np.zeros((3, 1), dtype=np.uint64)
    out = np.empty((3, 3))
    devs = (ctypes.c_int * 2)(0, 1)
    rc = lib.mi_all_pairs_host_devices(words.ctypes.data, 10, 3, 0, 1e-12, 1, 1, out.ctypes.data, None, 2)
    assert rc == nat.MI_ERR_DOMAIN and "devices" in nat.last_error()
    rc = lib.mi_all_pairs_host_devices(words.ctypes.data, 10, 3, 0, 1e-12, 1, 1, out.ctypes.data, devs, 0)
    assert rc == nat.MI_ERR_DOMAIN
    rc = lib.mi_all_pairs_host_devices(words.ctypes.data, 10, 3, 0, 1e-12, 1, 0, out.ctypes.data, devs, 2)
    assert rc == nat.MI_ERR_DOMAIN and "counts" in nat.last_error()
    rc = lib.mi_all_pairs_host_devices(words.ctypes.data, 0, 3, 0, 1e-12, 1, 1, out.ctypes.data, devs, 2)
    assert rc == nat.MI_ERR_DIMENSION
    dirty = np.array([[0b111]], dtype=np.uint64)  # padding bits set for n_rows = 2
    rc = lib.mi_all_pairs_host_devices(dirty.ctypes.data, 2, 1, 0, 1e-12, 1, 1, out.ctypes.data, devs, 2)
    assert rc == nat.MI_ERR_DOMAIN and "padding" in nat.last_error()


def test_tuning_knobs_roundtrip():
    old = nat.get_tuning("band")
    nat.set_tuning(band=4)
    assert nat.get_tuning("band") == 4
    nat.set_tuning(band=old)
    with pytest.raises(DomainError):
        nat.set_tuning(cta_group=3)
    with pytest.raises(DomainError):
        nat.set_tuning(nonsense=1)


# ------------------------------------------------------------------ data model
def test_binary_matrix_validation():
    """binmat.py:71-80 / test_binmat.py:101-104 semantics."""
    with pytest.raises(DimensionError):
        BinaryMatrix(0, 1, np.zeros((1, 0), dtype=np.uint64))
    with pytest.raises(DimensionError):
        BinaryMatrix(3, 2, np.zeros((2, 2), dtype=np.uint64))
    with pytest.raises(DomainError):
        BinaryMatrix(2, 1, np.array([[0b111]], dtype=np.uint64))
    with pytest.raises(DimensionError):
        from_rows([])
    with pytest.raises(DimensionError):
        from_rows([[1, 0], [1]])
    with pytest.raises(DomainError):
        from_rows([[0, 2]])
    m = from_rows([[1, 0], [0, 1], [1, 1]])
    assert m.words.tolist() == [[0b101], [0b110]]


@pytest.mark.parametrize("n", [1, 63, 64, 65, 128, 130])
def test_pack_matches_oracle(n):
    bits = rand_bits(np.random.default_rng(n), n, 5, 0.5)
    assert np.array_equal(from_bits(bits).words, O.pack_bits(bits))
    assert np.array_equal(from_bits(bits).to_bits(), bits)


def test_engine_config_and_backend_validation():
    with pytest.raises(DomainError):
        EngineConfig(mode="fuzzy")
    with pytest.raises(DomainError):
        EngineConfig(mode="epsilon", epsilon=0.0)
    assert BACKENDS == ("dense", "sparse", "direct")
    mat = from_rows([[1]])
    with pytest.raises(DomainError):
        mi_all_pairs(mat, backend="gpu")  # test_engine.py:152-154


def test_no_silent_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(NativeError):
        mi_all_pairs(from_rows([[1, 0], [0, 1]]))


# ------------------------------------------------------------------ datagen program
@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_product_recipe_agrees_with_oracle(cfg):
    n, m = {1: (1000, 500), 2: (3000, 600), 3: (100, 70), 4: (2000, 1000), 5: (400, 300)}[cfg]
    a = datagen.config_recipe(cfg, n, m)
    b = O.config_recipe(cfg, n, m)
    assert np.array_equal(a["density"], b["density"])
    assert a["zero_cols"] == b["zero_cols"] and a["one_cols"] == b["one_cols"]
    assert [tuple(p) for p in a["pairs"]] == [tuple(p) for p in b["pairs"]]
    thr, kind, src, ft = datagen.column_program(a)
    assert ((kind == 3).sum()) == len(a["pairs"])
    for c in a["zero_cols"]:
        assert kind[c] == 1
    assert datagen.threshold(0.5) == 1 << 63


def test_signature_binding_types():
    fn = nat.lib().mi_all_pairs_host
    assert fn.restype is ctypes.c_int and len(fn.argtypes) == 9


def test_staged_broadcast_plan():
    """Column groups of the staged broadcast: cover every block once, in
    order; auto_stages splits only long per-rank shares (host logic)."""
    from paper_2411_19702_b200 import dispatch

    for m in (1, 255, 256, 257, 10_000, 50_000):
        for S in (1, 2, 3, 4, 7):
            b = dispatch.stage_bounds(m, S)
            T = -(-m // 256)
            assert b[0][0] == 0 and b[-1][1] == T and b[-1][3] == m
            assert all(b[k][1] == b[k + 1][0] and b[k][3] == b[k + 1][2] for k in range(len(b) - 1))
            assert len(b) == min(S, T)
    assert dispatch.auto_stages(50_000, 1, 148) == 1
    assert dispatch.auto_stages(50_000, 8, 148) == 4     # config 4: ~33 rounds per rank
    assert dispatch.auto_stages(10_000, 8, 148) == 1     # config 3: ~1.4 rounds per rank
    assert dispatch.auto_stages(10_000, 2, 148) == 1


def test_every_documented_knob_round_trips():
    """Each knob the header documents is accepted, read back, and range-checked
    (host logic; no device needed)."""
    from paper_2411_19702_b200.errors import DomainError

    good = {"cta_group": 1, "prefetch": 4, "l2_hint": 0, "band": 3, "stages": 6, "epi_warps": 8, "fixed": 0,
            "table_thr": 1000, "pace": 16, "tail": 2, "fp4": 0, "evac": 2, "shard": 0, "hybrid": 1,
            "unperm_ctas": 2, "ingest": 6, "ingest_split": 1, "serp": 0, "xp_diag_w": 75}
    bad = {"ingest": 17, "ingest_split": 2, "serp": 2, "unperm_ctas": 5, "evac": 3, "tail": 4, "xp_diag_w": 5}
    old = {k: nat.get_tuning(k) for k in good}
    try:
        for k, v in good.items():
            nat.set_tuning(**{k: v})
            assert nat.get_tuning(k) == v, k
        for k, v in bad.items():
            with pytest.raises(DomainError):
                nat.set_tuning(**{k: v})
    finally:
        for k, v in old.items():
            nat.set_tuning(**{k: v})
