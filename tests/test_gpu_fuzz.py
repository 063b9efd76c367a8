"""Seeded fuzz over shapes, densities, EngineConfig variants, output types
and schedule knobs: every case bit-exact in counts and within the float64 /
float32 tolerance of the C oracle, bit-identically symmetric.  Shapes are
drawn to land on awkward tile counts (tail splits of every kind), ragged N
(e2m1 padding inside a 256-row k-block) and ragged m."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

KNOBS = [{}, {"tail": 2}, {"tail": 3}, {"tail": 0}, {"pace": 8}, {"fixed": 0}, {"fixed": 2},
         {"evac": 0}, {"evac": 2}, {"fp4": 0}, {"band": 1}, {"cta_group": 1}, {"fixed": 3}, {"hybrid": 0}]


def _case(k: int):
    rng = np.random.default_rng(1000 + k)
    n = int(rng.choice([1, 2, 63, 255, 256, 257, 511, 777, 1025, 2049, 4097]) + rng.integers(0, 3))
    m = int(rng.integers(1, 1600))
    dens = rng.choice([0.0, 0.02, 0.5, 0.97, 1.0], size=m, p=[0.05, 0.2, 0.5, 0.2, 0.05])
    dens = np.where(rng.random(m) < 0.5, rng.random(m), dens)
    bits = (rng.random((n, m)) < dens[None, :]).astype(np.uint8)
    if m > 4:
        bits[:, 1] = bits[:, 0]
        bits[:, 3] = 1 - bits[:, 2]
    mode = str(rng.choice(["exact", "exact", "epsilon"]))
    diag = bool(rng.random() < 0.8)
    dtype = str(rng.choice(["float64", "float64", "float32"]))
    knobs = KNOBS[k % len(KNOBS)]
    return n, m, O.pack_bits(bits), mode, diag, dtype, knobs


@pytest.mark.parametrize("k", range(48))
def test_fuzz_case(engine, k):
    from paper_2411_19702_b200 import EngineConfig
    from paper_2411_19702_b200 import _native as nat

    n, m, words, mode, diag, dtype, knobs = _case(k)
    cfg = EngineConfig(mode=mode, epsilon=1e-10, include_diagonal=diag)
    old = {key: nat.get_tuning(key) for key in knobs}
    try:
        nat.set_tuning(**knobs)
        dev = engine.upload(words)
        g, v = engine.gram_counts(dev, n, m)
        mi = engine.all_pairs_device(engine.upload(words), n, m, cfg, getattr(torch, dtype)).cpu().numpy()
    finally:
        nat.set_tuning(**old)
    assert np.array_equal(g.cpu().numpy().astype(np.int64), O.c_gram_ones(words)), (n, m, knobs)
    assert np.array_equal(v.cpu().numpy().astype(np.uint64), O.c_column_sums(words))
    ref = O.c_mi_all_pairs(words, n, mode=mode, epsilon=1e-10, include_diagonal=diag)
    assert np.array_equal(mi, mi.T)
    tol = 1e-12 if dtype == "float64" else 1e-6
    err = float(np.max(np.abs(mi.astype(np.float64) - ref)))
    assert err < tol, (n, m, mode, diag, dtype, knobs, err)


@pytest.mark.parametrize("k", range(24))
def test_fuzz_new_paths(engine, k):
    """The same random cases through the column-sum order, the staged host
    path (random group count, pageable or pinned words) and the device packer:
    counts bit-exact, MI within tolerance, host path bit-identical to the
    device path."""
    from paper_2411_19702_b200 import EngineConfig
    from paper_2411_19702_b200 import _native as nat

    n, m, words, mode, diag, dtype, _ = _case(100 + k)
    rng = np.random.default_rng(5000 + k)
    cfg = EngineConfig(mode=mode, epsilon=1e-10, include_diagonal=diag)
    dt = getattr(torch, dtype)
    tol = 1e-12 if dtype == "float64" else 1e-6
    ref = O.c_mi_all_pairs(words, n, mode=mode, epsilon=1e-10, include_diagonal=diag)
    bits = O.unpack_bits(words, n)
    dev = engine.pack_bits(torch.from_numpy(bits).to(engine.device))
    assert np.array_equal(dev.cpu().numpy().view(np.uint64), words)
    # column-sum order
    got = engine.all_pairs_device(dev, n, m, cfg, dt, order="colsum").double().cpu().numpy()
    assert np.array_equal(got, got.T)
    assert float(np.max(np.abs(got - ref))) < tol, (n, m, "colsum")
    prep = engine.prepare(dev, n, m, order="colsum")
    g = engine.compute(prep, None, torch.int32).cpu().numpy().astype(np.int64)
    assert np.array_equal(g, O.c_gram_ones(words))
    # staged host path vs the device path
    natural = engine.all_pairs_device(dev, n, m, cfg, dt).cpu().numpy()
    old = nat.get_tuning("ingest")
    try:
        nat.set_tuning(ingest=int(rng.integers(0, 9)))
        src = torch.from_numpy(words.view(np.int64)).pin_memory() if rng.random() < 0.5 else words
        host = np.asarray(engine.all_pairs_host(src, n, m, cfg, dt))
    finally:
        nat.set_tuning(ingest=old)
    assert np.array_equal(host, natural)
