"""Pin the CPU oracle to the real reference (CPU only).

tests/golden/ holds the reference's own outputs (column_sums, gram_ones,
gram_complete_optimized, mi_all_pairs in exact / epsilon / no-diagonal
modes, datagen streams), recorded by golden/make_golden.py which imports
/root/reference.  Both restatements -- NumPy (oracle/oracle.py) and C
(oracle/mi_oracle.c) -- must reproduce them: counts bit-exact, NumPy MI
bit-identical (same operations), C MI within 1e-13.
"""

from __future__ import annotations

import hashlib
import math

import numpy as np
import pytest

from conftest import rand_bits
from oracle import oracle as O


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _cases(golden):
    arrays, meta = golden
    for name, case in meta["cases"].items():
        yield name, case, arrays


def test_counts_match_reference(golden):
    for name, case, arrays in _cases(golden):
        words = arrays[f"{name}/words"]
        v = O.column_sums(words)
        assert np.array_equal(v, arrays[f"{name}/v"]), name
        assert np.array_equal(O.c_column_sums(words), v), name
        g = O.gram_ones(words)
        assert sha(g) == case["g11_sha256"], name
        assert np.array_equal(O.c_gram_ones(words), g), name
        _, g00, g01 = O.gram_complete_optimized(g, v, case["n_rows"])
        assert sha(g00) == case["g00_sha256"] and sha(g01) == case["g01_sha256"], name


def test_mi_matches_reference(golden):
    for name, case, arrays in _cases(golden):
        words, n = arrays[f"{name}/words"], case["n_rows"]
        mi_np = O.mi_all_pairs(words, n)
        mi_c = O.c_mi_all_pairs(words, n)
        if case["full"]:
            ref = arrays[f"{name}/mi"]
            got_np, got_c = mi_np, mi_c
        else:
            ii, jj = arrays[f"{name}/sample_i"], arrays[f"{name}/sample_j"]
            ref, got_np, got_c = arrays[f"{name}/sample_mi"], mi_np[ii, jj], mi_c[ii, jj]
        assert np.array_equal(got_np, ref), f"{name}: NumPy restatement not bit-identical"
        assert float(np.max(np.abs(got_c - ref))) < 1e-13, name
        assert abs(mi_np.sum() - case["mi_checksum"]) < 1e-9


def test_mi_variants_match_reference(golden):
    for name, case, arrays in _cases(golden):
        for var in case["variants"]:
            words, n = arrays[f"{name}/words"], case["n_rows"]
            mi = O.mi_all_pairs(words, n, var["mode"], var["epsilon"], var["include_diagonal"])
            mc = O.c_mi_all_pairs(words, n, var["mode"], var["epsilon"], var["include_diagonal"])
            ref = arrays[f"{name}/mi_{var['name']}"]
            if not case["full"]:
                ii, jj = arrays[f"{name}/sample_i"], arrays[f"{name}/sample_j"]
                mi, mc = mi[ii, jj], mc[ii, jj]
            assert np.array_equal(mi, ref), f"{name}/{var['name']}"
            assert float(np.max(np.abs(mc - ref))) < 1e-13


def test_naive_oracle_matches_reference(golden):
    for name, case, arrays in _cases(golden):
        key = f"{name}/mi_naive"
        if key not in arrays.files:
            continue
        bits = O.unpack_bits(arrays[f"{name}/words"], case["n_rows"])
        m = bits.shape[1]
        for i in range(m):
            for j in range(i, m):
                assert abs(O.mi_pairwise_naive(bits[:, i], bits[:, j]) - arrays[key][i, j]) < 1e-15


def test_known_answers():
    """test_engine.py:25,36-41,74-93 and test_gram.py:21-22,39-43."""
    assert O.mi_pairwise_naive([0, 1, 0, 1], [0, 1, 0, 1]) == 1.0
    assert O.mi_pairwise_naive([0, 0, 1, 1], [0, 1, 0, 1]) == 0.0
    assert abs(O.mi_pairwise_naive([0, 0, 1, 1], [0, 1, 1, 1]) - 0.311278124459133) < 1e-12
    assert abs(O.binary_entropy(0.75) - 0.811278124459133) < 1e-12
    w = O.pack_bits(np.array([[1, 0], [0, 1], [1, 1]], dtype=np.uint8))
    g = O.gram_ones(w)
    assert g.tolist() == [[2, 1], [1, 2]]
    _, g00, g01 = O.gram_complete_optimized(g, O.column_sums(w), 3)
    assert g00.tolist() == [[1, 0], [0, 1]] and g01.tolist() == [[0, 1], [1, 0]]
    bal = O.mi_all_pairs(O.pack_bits(np.array([[0, 0], [1, 1], [0, 0], [1, 1]], np.uint8)), 4)
    assert bal[0, 1] == 1.0
    # bit layout: rows 0 and 64 -> words[0,0] = 1, words[0,1] = 1 (test_binmat.py:92-99)
    b = np.zeros((65, 1), dtype=np.uint8)
    b[0, 0] = b[64, 0] = 1
    assert O.pack_bits(b).tolist() == [[1, 1]]


def test_consistency_checks():
    """gram.py:98-110 -- corrupted inputs are rejected (test_gram.py:57-67)."""
    g = np.array([[2, 1], [1, 2]], dtype=np.int64)
    v = np.array([2, 2], dtype=np.uint64)
    with pytest.raises(O.OracleError):
        O.gram_complete_optimized(np.array([[2, 1], [0, 2]]), v, 3)
    with pytest.raises(O.OracleError):
        O.gram_complete_optimized(g, np.array([2, 1], dtype=np.uint64), 3)
    with pytest.raises(O.OracleError):
        O.gram_complete_optimized(g, v, 1)


def test_identity_theorem_small():
    """Closed-form counts equal direct four-cell counting (test_acceptance.py:53-82)."""
    rng = np.random.default_rng(2024)
    for n, m, d in [(1, 1, 0.5), (1, 64, 0.5), (64, 1, 0.0), (65, 2, 1.0), (130, 17, 0.3)]:
        bits = rand_bits(rng, n, m, d)
        w = O.pack_bits(bits)
        g11, g00, g01 = O.gram_complete_optimized(O.gram_ones(w), O.column_sums(w), n)
        b = bits.astype(np.int64)
        assert np.array_equal(g11, b.T @ b)
        assert np.array_equal(g00, (1 - b).T @ (1 - b))
        assert np.array_equal(g01, (1 - b).T @ b)


def test_datagen_streams_match_reference(golden):
    arrays, meta = golden
    for key in arrays.files:
        if not key.startswith("datagen/gen_"):
            continue
        parts = key.split("_")
        n, m = map(int, parts[1].split("x"))
        seed, dens = int(parts[2][1:]), float(parts[3][1:])
        assert np.array_equal(O.pack_bits(O.generate_bits(n, m, dens, seed)), arrays[key]), key
    w1 = O.pack_bits(O.generate_bits(1000, 500, 0.5, 0))
    assert sha(w1) == meta["datagen"]["cfg1"]["words_sha256"]
    rec = O.config_recipe(1)
    assert rec["zero_cols"] + rec["one_cols"] == meta["cfg1_planted_columns"]
    assert sha(O.gram_ones(O.pack_bits(O.generate_config_bits(rec)))) == \
        meta["cases"]["cfg1_planted"]["g11_sha256"]


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_c_generator_matches_numpy(cfg):
    n, m = {1: (1000, 500), 2: (3000, 600), 3: (130, 70), 4: (2000, 1000), 5: (400, 300)}[cfg]
    rec = O.config_recipe(cfg, n, m)
    full = O.pack_bits(O.generate_config_bits(rec))
    assert np.array_equal(O.c_generate_config_words(rec), full)
    cols = [0, m - 1] + [t for _, t in rec["pairs"][:3]] + [s for s, _ in rec["pairs"][:3]]
    assert np.array_equal(O.c_generate_config_words(rec, cols), full[cols])
    assert np.array_equal(O.pack_bits(O.generate_config_columns(rec, cols)), full[cols])


def test_cfg3_digest_matches_reference(golden):
    """The C generator reproduces the reference's generate(GenSpec(1e5, 1e4, .5, 2))."""
    _, meta = golden
    if "cfg3" not in meta["datagen"]:
        pytest.skip("cfg3 digest not recorded")
    d = meta["datagen"]["cfg3"]
    rec = O.config_recipe(3)
    sub = meta["cfg3_subset_columns"]
    w = O.c_generate_config_words(rec, sub)
    assert [int(x) for x in w[0, :4]] == d["words_head"]
    assert [int(x) for x in w[-1, -4:]] == d["words_tail"]


def test_cfg3_subset_parity(golden):
    arrays, meta = golden
    if "cfg3_subset" not in meta["cases"]:
        pytest.skip("cfg3 subset not recorded")
    w = O.c_generate_config_words(O.config_recipe(3), meta["cfg3_subset_columns"])
    assert np.array_equal(w, arrays["cfg3_subset/words"])


def test_entropy_diagonal_property():
    rng = np.random.default_rng(43)
    bits = rand_bits(rng, 130, 10, 0.25)
    mi = O.mi_all_pairs(O.pack_bits(bits), 130)
    for j in range(10):
        p = bits[:, j].mean()
        assert abs(mi[j, j] - O.binary_entropy(p)) < 1e-12
    assert math.isfinite(mi.sum())
