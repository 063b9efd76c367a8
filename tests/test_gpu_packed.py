"""Egress: the packed upper-triangle output (MI_PACKED_UPPER:
row i holds columns i..m-1, m(m+1)/2 elements) through the device API and the
streamed host API is exactly the upper triangle of the full result."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import rand_bits
from oracle import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("n,m", [(1, 1), (100, 7), (777, 300), (4_097, 1_300), (5_000, 3_000), (20_000, 700)])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_packed_equals_upper_triangle(engine, n, m, dtype):
    from paper_2411_19702_b200.engine import unpack_upper

    rng = np.random.default_rng(n * 3 + m)
    words = O.pack_bits(rand_bits(rng, n, m, 0.4))
    dt = getattr(torch, dtype)
    dev = engine.upload(words)
    full = engine.all_pairs_device(dev, n, m, None, dt).cpu().numpy()
    prep = engine.prepare(dev, n, m)
    packed = engine.compute(prep, None, dt, packed=True).cpu().numpy()
    iu = np.triu_indices(m)
    assert np.array_equal(packed, full[iu])
    assert np.array_equal(unpack_upper(packed, m), full)
    host = np.asarray(engine.all_pairs_host(words, n, m, None, dt, packed=True))
    assert np.array_equal(host, full[iu])


@pytest.mark.parametrize("ingest", [0, 1, 2, 3, 4, 16])
@pytest.mark.parametrize("n,m", [(100, 7), (777, 300), (4_097, 1_300), (3_000, 2_600), (20_000, 700)])
def test_staged_host_path_equals_device(engine, ingest, n, m):
    """mi_all_pairs_host with S staged column groups (upload, unpack, the
    group's tiles, 2-D egress of the region they complete) or the row-band
    path (ingest 0): bit-identical to the device path, both dtypes."""
    from paper_2411_19702_b200 import _native as nat

    rng = np.random.default_rng(n + 7 * m)
    dens = rng.uniform(0.01, 0.99, m)
    words = O.pack_bits((rng.random((n, m)) < dens[None, :]).astype(np.uint8))
    dev = engine.upload(words)
    old = nat.get_tuning("ingest")
    try:
        nat.set_tuning(ingest=ingest)
        for dt in (torch.float64, torch.float32):
            full = engine.all_pairs_device(dev, n, m, None, dt).cpu().numpy()
            pinned = torch.empty((m, m), dtype=dt, pin_memory=True)
            host = engine.all_pairs_host(words, n, m, None, dt, host_out=pinned).numpy()
            assert np.array_equal(host, full)
            pageable = engine.all_pairs_host(words, n, m, None, dt, host_out=torch.empty((m, m), dtype=dt)).numpy()
            assert np.array_equal(pageable, full)
            fresh = engine.all_pairs_host(words, n, m, None, dt)  # default: a fresh numpy array
            assert isinstance(fresh, np.ndarray) and np.array_equal(fresh, full)
    finally:
        nat.set_tuning(ingest=old)


def test_config3_host_path_full_size(engine):
    """The e2e path at its bench size: config 3 (N = 100,000 x m = 10,000,
    float64) through mi_all_pairs_host -- staged upload / compute / download,
    pageable numpy words in (host-thread staging), a fresh pageable numpy
    output (the pinned egress buffer) -- bit-identical to the device path,
    and through the drop-in mi_all_pairs."""
    from paper_2411_19702_b200 import BinaryMatrix, datagen, mi_all_pairs

    rec = datagen.config_recipe(3)
    n, m = rec["n"], rec["m"]
    dev = datagen.generate_words_device(rec, engine.device)
    full = engine.all_pairs_device(dev, n, m).cpu().numpy()
    words = dev.cpu().numpy().view(np.uint64)
    host = engine.all_pairs_host(words, n, m)
    assert isinstance(host, np.ndarray) and host.dtype == np.float64
    assert np.array_equal(host, full)
    res = mi_all_pairs(BinaryMatrix(n, m, words))
    assert res.values.flags.c_contiguous and res.values.flags.owndata
    assert np.array_equal(res.values, full)
