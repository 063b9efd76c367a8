"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference's golden outputs.

Bar (BASELINE.json / SURVEY 8(c)): co-occurrence counts bit-exact; MI within
1e-6 absolute of the reference's float64 result (the float64 path is held to
1e-12 here, the same tolerance the reference's own tests use); exact 1.0 /
0.0 golden values reproduced exactly; output bit-identically symmetric.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import rand_bits
from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

TOL_F64 = 1e-12   # reference's own tolerance for bulk-vs-oracle (test_engine.py:121-140)
TOL_F32 = 1e-6    # BASELINE contract for the float32 device output


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gpu_counts(engine, words, n):
    m = words.shape[0]
    g, v = engine.gram_counts(engine.upload(words), n, m)
    return g.cpu().numpy().astype(np.int64), v.cpu().numpy().astype(np.uint64)


def gpu_mi(engine, words, n, cfg=None, dtype=None):
    dtype = dtype or torch.float64
    m = words.shape[0]
    out = engine.all_pairs_device(engine.upload(words), n, m, cfg, dtype)
    return out.cpu().numpy()


def cfg_of(mode="exact", eps=1e-12, diag=True):
    from paper_2411_19702_b200 import EngineConfig

    return EngineConfig(mode=mode, epsilon=eps, include_diagonal=diag)


# --------------------------------------------------------------- golden cases

def test_counts_bit_exact_on_golden(engine, golden):
    arrays, meta = golden
    for name, case in meta["cases"].items():
        words = arrays[f"{name}/words"]
        g, v = gpu_counts(engine, words, case["n_rows"])
        assert np.array_equal(v, arrays[f"{name}/v"]), f"{name}: column sums"
        assert sha(g) == case["g11_sha256"], f"{name}: G11 differs from reference gram_ones"


def test_mi_f64_matches_reference_on_golden(engine, golden):
    arrays, meta = golden
    worst = 0.0
    for name, case in meta["cases"].items():
        words = arrays[f"{name}/words"]
        mi = gpu_mi(engine, words, case["n_rows"])
        assert mi.dtype == np.float64 and mi.shape == (case["n_cols"],) * 2
        assert np.array_equal(mi, mi.T), f"{name}: not bit-identically symmetric"
        if case["full"]:
            ref = arrays[f"{name}/mi"]
            got = mi
        else:
            ii, jj = arrays[f"{name}/sample_i"], arrays[f"{name}/sample_j"]
            ref, got = arrays[f"{name}/sample_mi"], mi[ii, jj]
        err = float(np.max(np.abs(got - ref)))
        worst = max(worst, err)
        assert err < TOL_F64, f"{name}: max |gpu - ref| = {err}"
        assert abs(mi.sum() - case["mi_checksum"]) < 1e-9 * max(1.0, case["n_cols"] ** 2)
    print(f"worst |gpu - reference| over golden cases: {worst:.3e}")


def test_mi_variants_on_golden(engine, golden):
    arrays, meta = golden
    for name, case in meta["cases"].items():
        for var in case["variants"]:
            cfg = cfg_of(var["mode"], var["epsilon"], var["include_diagonal"])
            mi = gpu_mi(engine, arrays[f"{name}/words"], case["n_rows"], cfg)
            ref = arrays[f"{name}/mi_{var['name']}"]
            got = mi if case["full"] else mi[arrays[f"{name}/sample_i"], arrays[f"{name}/sample_j"]]
            err = float(np.max(np.abs(got - ref)))
            assert err < TOL_F64, f"{name}/{var['name']}: {err}"
            if not var["include_diagonal"]:
                assert np.all(np.diagonal(mi) == 0.0)


def test_golden_values_exact(engine, golden):
    """test_acceptance.py:112-125 / test_engine.py:25,74-93 through the GPU path."""
    arrays, _ = golden
    bal = gpu_mi(engine, arrays["balanced_identical/words"], 4)
    assert bal[0, 1] == 1.0 and bal[1, 0] == 1.0
    ind = gpu_mi(engine, arrays["independent/words"], 4)
    assert ind[0, 1] == 0.0
    gold = gpu_mi(engine, arrays["golden_0011_0111/words"], 4)
    assert abs(gold[0, 1] - 0.311278124459133) < 1e-12
    h = gpu_mi(engine, arrays["h075/words"], 4)
    assert abs(h[0, 0] - 0.811278124459133) < 1e-12
    one_row = gpu_mi(engine, arrays["single_row/words"], 1)
    assert np.all(one_row == 0.0)


def test_f32_output_within_contract(engine, golden):
    arrays, meta = golden
    for name, case in meta["cases"].items():
        mi = gpu_mi(engine, arrays[f"{name}/words"], case["n_rows"], None, torch.float32)
        assert mi.dtype == np.float32
        ref = arrays[f"{name}/mi"] if case["full"] else arrays[f"{name}/sample_mi"]
        got = mi if case["full"] else mi[arrays[f"{name}/sample_i"], arrays[f"{name}/sample_j"]]
        assert float(np.max(np.abs(got.astype(np.float64) - ref))) < TOL_F32, name


# --------------------------------------------------------------- edge shapes

EDGE_SHAPES = [
    (1, 1), (1, 300), (2, 257), (63, 255), (64, 256), (65, 257), (127, 511), (128, 512),
    (129, 513), (255, 300), (256, 129), (1000, 700), (3000, 1025),
]


@pytest.mark.parametrize("n,m", EDGE_SHAPES)
@pytest.mark.parametrize("density", [0.0, 0.3, 1.0])
def test_edge_shapes_counts_and_mi(engine, n, m, density):
    rng = np.random.default_rng(n * 7919 + m + int(density * 10))
    bits = rand_bits(rng, n, m, density)
    words = O.pack_bits(bits)
    g, v = gpu_counts(engine, words, n)
    assert np.array_equal(v, O.column_sums(words))
    assert np.array_equal(g, O.c_gram_ones(words))
    mi = gpu_mi(engine, words, n)
    ref = O.c_mi_all_pairs(words, n)
    assert np.array_equal(mi, mi.T)
    assert float(np.max(np.abs(mi - ref))) < TOL_F64


KNOB_VARIANTS = [
    {"pace": 0}, {"pace": 1}, {"pace": 16}, {"pace": 100000}, {"cta_group": 1}, {"cta_group": 1, "pace": 16},
    {"fixed": 0}, {"fixed": 2}, {"band": 1}, {"band": 3}, {"l2_hint": 0}, {"prefetch": 4},
    {"tail": 0}, {"tail": 0, "pace": 16}, {"tail": 0, "cta_group": 1},
    {"tail": 2}, {"tail": 3}, {"tail": 3, "cta_group": 1}, {"tail": 2, "cta_group": 1}, {"tail": 3, "pace": 16},
    {"fp4": 0}, {"fp4": 0, "tail": 3}, {"fp4": 0, "pace": 16}, {"fp4": 0, "fixed": 0},
    {"fixed": 3}, {"hybrid": 0}, {"fixed": 3, "fp4": 0}, {"serp": 0}, {"serp": 0, "pace": 16}, {"serp": 1},
    {"xp": 0}, {"xp": 1}, {"xp": 1, "tail": 3}, {"xp": 1, "tail": 2}, {"xp": 1, "fixed": 0}, {"xp": 1, "evac": 0},
]


@pytest.mark.parametrize("tail", [0, 2, 3])
@pytest.mark.parametrize("n,m", [(3000, 3000), (700, 9700), (5000, 768)])
def test_tail_split_shapes(engine, tail, n, m):
    """Tile counts with 1-6 tiles in the last round (78, 741, 6 tiles at 256):
    column-slice and K-range tails agree with the untouched schedule bit for
    bit (integer counts, and MI computed from the same counts), through the
    device API and the streamed host API."""
    from paper_2411_19702_b200 import BinaryMatrix, mi_all_pairs_c_abi
    from paper_2411_19702_b200 import _native as nat

    rng = np.random.default_rng(n + m)
    bits = rand_bits(rng, n, m, 0.45)
    words = O.pack_bits(bits)
    old = nat.get_tuning("tail")
    try:
        nat.set_tuning(tail=0)
        ref_g, _ = gpu_counts(engine, words, n)
        ref_mi = gpu_mi(engine, words, n)
        nat.set_tuning(tail=tail)
        g, _ = gpu_counts(engine, words, n)
        mi = gpu_mi(engine, words, n)
        host = mi_all_pairs_c_abi(BinaryMatrix(n, m, words))
    finally:
        nat.set_tuning(tail=old)
    assert np.array_equal(g, ref_g)
    assert np.array_equal(mi, ref_mi)
    assert np.array_equal(host, ref_mi)
    if m <= 3000:
        assert np.array_equal(g, O.c_gram_ones(words))


@pytest.mark.parametrize("knobs", KNOB_VARIANTS, ids=lambda k: ",".join(f"{a}={b}" for a, b in k.items()))
def test_tuning_variants_agree(engine, knobs):
    """Every tuning knob (tile size, L2 pacing, epilogue path, tile order, L2
    hints) changes the schedule only: counts stay bit-exact and MI within the
    float64 tolerance of the oracle."""
    from paper_2411_19702_b200 import _native as nat

    rng = np.random.default_rng(4242)
    n, m = 20_000, 1_100
    bits = rand_bits(rng, n, m, 0.3)
    words = O.pack_bits(bits)
    old = {k: nat.get_tuning(k) for k in knobs}
    try:
        nat.set_tuning(**knobs)
        g, v = gpu_counts(engine, words, n)
        mi = gpu_mi(engine, words, n)
    finally:
        nat.set_tuning(**old)
    assert np.array_equal(g, O.c_gram_ones(words))
    ref = O.c_mi_all_pairs(words, n)
    assert np.array_equal(mi, mi.T)
    assert float(np.max(np.abs(mi - ref))) < TOL_F64


def test_determinism_and_c_abi_host_path(engine):
    from paper_2411_19702_b200 import BinaryMatrix, mi_all_pairs, mi_all_pairs_c_abi

    rng = np.random.default_rng(99)
    bits = rand_bits(rng, 2000, 600, 0.4)
    mat = BinaryMatrix(2000, 600, O.pack_bits(bits))
    a = mi_all_pairs(mat).values
    b = mi_all_pairs(mat, threads=1).values
    c = mi_all_pairs_c_abi(mat)
    assert np.array_equal(a, b) and np.array_equal(a, c)
    assert a.flags["C_CONTIGUOUS"] and a.dtype == np.float64


def test_backends_and_errors(engine):
    from paper_2411_19702_b200 import BinaryMatrix, DomainError, EngineConfig, mi_all_pairs

    rng = np.random.default_rng(5)
    mat = BinaryMatrix(100, 9, O.pack_bits(rand_bits(rng, 100, 9, 0.5)))
    dense = mi_all_pairs(mat, backend="dense").values
    for b in ("sparse", "direct"):
        assert np.array_equal(mi_all_pairs(mat, backend=b).values, dense)
    with pytest.raises(DomainError):
        mi_all_pairs(mat, backend="gpu")
    with pytest.raises(DomainError):
        EngineConfig(mode="fuzzy")


# --------------------------------------------------------------- generator

def test_generator_bit_exact(engine, golden):
    from paper_2411_19702_b200 import datagen

    arrays, meta = golden
    for key in arrays.files:
        if not key.startswith("datagen/gen_"):
            continue
        parts = key.split("_")
        n, m = map(int, parts[1].split("x"))
        seed, dens = int(parts[2][1:]), float(parts[3][1:])
        w = datagen.generate(n, m, dens, seed, engine.device).cpu().numpy().view(np.uint64)
        assert np.array_equal(w, arrays[key]), key
    w1 = datagen.generate(1000, 500, 0.5, 0, engine.device).cpu().numpy().view(np.uint64)
    assert sha(w1) == meta["datagen"]["cfg1"]["words_sha256"]


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_config_recipes_bit_exact(engine, cfg):
    from paper_2411_19702_b200 import datagen

    n, m = {1: (1000, 500), 2: (3000, 600), 3: (700, 300), 4: (2000, 1000), 5: (4000, 300)}[cfg]
    rec = datagen.config_recipe(cfg, n, m)
    w = datagen.generate_words_device(rec, engine.device).cpu().numpy().view(np.uint64)
    ref = O.pack_bits(O.generate_config_bits(O.config_recipe(cfg, n, m)))
    assert np.array_equal(w, ref)


def _stress_words(n, m, seed):
    """Columns that stress the float32 epilogue: densities from 1e-4 to
    1 - 1e-4, exact copies, complements, subsets and near-copies."""
    rng = np.random.default_rng(seed)
    dens = np.concatenate([[1e-4, 1e-3, 0.01, 0.5, 0.99, 0.999, 0.9999], rng.uniform(0, 1, m)])[:m]
    bits = (rng.random((n, m)) < dens[None, :]).astype(np.uint8)
    for k in range(0, m - 8, 23):
        bits[:, k + 1] = bits[:, k]                                  # copy
        bits[:, k + 2] = 1 - bits[:, k]                              # complement
        bits[:, k + 3] = bits[:, k] & (rng.random(n) < 0.5)          # subset
        bits[:, k + 4] = bits[:, k] ^ (rng.random(n) < 0.001)        # near copy
    return O.pack_bits(bits)


@pytest.mark.parametrize("n,m", [(20_000, 700), (1_000, 300), (300_000, 260), (4_097, 513)])
@pytest.mark.parametrize("fixed", [0, 1])
def test_f32_epilogue_stress(engine, n, m, fixed):
    """float32 output (fixed=0: the FP64 epilogue on every tile; 1 = adaptive,
    table path where the column sums allow) stays within the 1e-6 contract of
    the float64 oracle on adversarial columns, bit-identically symmetric."""
    from paper_2411_19702_b200 import _native as nat

    words = _stress_words(n, m, seed=n + m)
    old = nat.get_tuning("fixed")
    try:
        nat.set_tuning(fixed=fixed)
        mi = gpu_mi(engine, words, n, None, torch.float32)
    finally:
        nat.set_tuning(fixed=old)
    ref = O.c_mi_all_pairs(words, n)
    assert np.array_equal(mi, mi.T)
    err = float(np.max(np.abs(mi.astype(np.float64) - ref)))
    assert err < TOL_F32, err


def test_concurrent_streams_with_k_range_tails(engine):
    """Two host threads launch on two streams at once; both shapes use the
    K-range tail (shared per-device partial slots), which the C ABI chains
    across streams: every result equals its serial result."""
    import threading

    from paper_2411_19702_b200 import _native as nat

    shapes = [(40_000, 3000, 1), (30_000, 3000, 2)]  # 78 tiles: 4 tail tiles, K-range split
    data = []
    for n, m, seed in shapes:
        words = O.pack_bits(rand_bits(np.random.default_rng(seed), n, m, 0.4))
        dev = engine.upload(words)
        data.append((n, m, dev, engine.all_pairs_device(dev, n, m).cpu().numpy()))
    assert nat.get_tuning("tail") in (1, 3)
    results = [None, None]

    def work(k):
        n, m, dev, _ = data[k]
        s = torch.cuda.Stream(engine.device)
        with torch.cuda.stream(s):
            outs = [engine.all_pairs_device(dev, n, m) for _ in range(6)]
        s.synchronize()
        results[k] = [o.cpu().numpy() for o in outs]

    threads = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for k in range(2):
        for got in results[k]:
            assert np.array_equal(got, data[k][3])


@pytest.mark.parametrize("mode,diag,dtype", [("exact", False, "float64"), ("epsilon", True, "float64"),
                                             ("epsilon", False, "float32"), ("exact", True, "float32")])
def test_config_variants_with_full_rounds(engine, mode, diag, dtype):
    """m = 3000 (78 tiles: a full round of 74 pairs, so main-loop tiles run
    the evacuated epilogue, plus a split tail) in every EngineConfig variant."""
    n, m = 5_000, 3_000
    rng = np.random.default_rng(31)
    words = O.pack_bits(rand_bits(rng, n, m, 0.5))
    dt = getattr(torch, dtype)
    mi = gpu_mi(engine, words, n, cfg_of(mode, 1e-9, diag), dt)
    ref = O.c_mi_all_pairs(words, n, mode=mode, epsilon=1e-9, include_diagonal=diag)
    assert np.array_equal(mi, mi.T)
    tol = TOL_F64 if dtype == "float64" else TOL_F32
    assert float(np.max(np.abs(mi.astype(np.float64) - ref))) < tol
    if not diag:
        assert np.all(np.diagonal(mi) == 0)


def test_serpentine_k_order_is_bit_identical(engine):
    """serp = 1 sweeps K backwards on odd tile rounds (>= 2 rounds here: 136
    tiles on 74 SM pairs); counts and MI match the forward order bit for bit."""
    from paper_2411_19702_b200 import _native as nat

    rng = np.random.default_rng(77)
    n, m = 5_000, 4_000
    dens = rng.uniform(0.02, 0.98, m)
    words = O.pack_bits((rng.random((n, m)) < dens[None, :]).astype(np.uint8))
    res = {}
    old = nat.get_tuning("serp")
    for sp in (0, 1):
        nat.set_tuning(serp=sp)
        try:
            res[sp] = (gpu_counts(engine, words, n)[0], gpu_mi(engine, words, n))
        finally:
            nat.set_tuning(serp=old)
    assert np.array_equal(res[0][0], res[1][0])
    assert np.array_equal(res[0][1], res[1][1])
    assert np.array_equal(res[1][0], O.c_gram_ones(words))


def test_invariants_like_the_reference(engine):
    """test_engine.py:157-219's invariant suite through the GPU path: row
    permutation leaves the matrix bit-identical (the counts are identical),
    complementing a column or duplicating every row changes MI by < 1e-12,
    0 <= MI(i, j) <= min(H_i, H_j), epsilon mode within 1e-6 of exact."""
    rng = np.random.default_rng(2024)
    n, m = 3000, 700
    dens = rng.uniform(0.05, 0.95, m)
    bits = (rng.random((n, m)) < dens[None, :]).astype(np.uint8)
    base = gpu_mi(engine, O.pack_bits(bits), n)
    perm = rng.permutation(n)
    assert np.array_equal(gpu_mi(engine, O.pack_bits(bits[perm]), n), base)
    comp = bits.copy()
    comp[:, 5] = 1 - comp[:, 5]
    assert float(np.max(np.abs(gpu_mi(engine, O.pack_bits(comp), n) - base))) < 1e-12
    dup = np.concatenate([bits, bits], axis=0)
    assert float(np.max(np.abs(gpu_mi(engine, O.pack_bits(dup), 2 * n) - base))) < 1e-12
    h = np.diagonal(base)
    assert base.min() >= -1e-12
    assert float(np.max(base - np.minimum(h[:, None], h[None, :]))) <= 1e-12
    eps = gpu_mi(engine, O.pack_bits(bits), n, cfg_of("epsilon", 1e-12))
    assert float(np.max(np.abs(eps - base))) <= 1e-6
