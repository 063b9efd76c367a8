"""Several GPUs in one process (mi_all_pairs_host_devices / the drop-in's
``devices=``): the triangle's tiles dealt as over the multi-GPU path's
ranks, every device writing its tiles and mirrors into the host matrix.  On
the one-GPU box the same device is listed several times (each listing runs
one share on its own stream); results must equal one device's bit for bit
(/root/reference/pkg/src/mimatrix/engine.py:137-138: one symmetric matrix)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import rand_bits
from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.mark.parametrize("n,m,d", [(20_000, 700, 0.3), (6_000, 3_300, 0.5), (300, 9, 0.5), (50_000, 2_100, 0.05)])
@pytest.mark.parametrize("k", [2, 3, 8])
def test_devices_equal_one_device(engine, n, m, d, k):
    from paper_2411_19702_b200 import BinaryMatrix, EngineConfig, mi_all_pairs, mi_all_pairs_devices

    rng = np.random.default_rng(n + m + k)
    mat = BinaryMatrix(n, m, O.pack_bits(rand_bits(rng, n, m, d)))
    one = mi_all_pairs(mat).values
    many = mi_all_pairs(mat, devices=[0] * k).values
    assert np.array_equal(one, many)
    f32 = mi_all_pairs_devices(mat, [0] * k, out_dtype=np.float32)
    assert np.array_equal(f32, engine.all_pairs_host(mat.words, n, m, None, torch.float32))
    cfg = EngineConfig(mode="epsilon", epsilon=1e-9, include_diagonal=False)
    assert np.array_equal(mi_all_pairs_devices(mat, [0] * k, cfg), mi_all_pairs(mat, cfg).values)


def test_devices_into_registered_output(engine):
    """A pinned, mapped output is written zero-copy by every device."""
    from paper_2411_19702_b200 import BinaryMatrix, mi_all_pairs, mi_all_pairs_devices
    from paper_2411_19702_b200 import _native as nat

    n, m = 40_000, 1_500
    rng = np.random.default_rng(12)
    mat = BinaryMatrix(n, m, O.pack_bits(rand_bits(rng, n, m, 0.4)))
    out = np.empty((m, m), dtype=np.float64)
    nat.check(nat.lib().mi_host_register(out.ctypes.data, out.nbytes), "mi_host_register")
    try:
        mi_all_pairs_devices(mat, [0, 0, 0, 0], out=out)
    finally:
        nat.lib().mi_host_unregister(out.ctypes.data)
    assert np.array_equal(out, mi_all_pairs(mat).values)
    assert np.max(np.abs(out - O.c_mi_all_pairs(mat.words, n))) < 1e-12


def test_devices_reject_bad_lists(engine):
    from paper_2411_19702_b200 import BinaryMatrix, DomainError, NativeError, mi_all_pairs_devices

    mat = BinaryMatrix(100, 5, O.pack_bits(rand_bits(np.random.default_rng(0), 100, 5, 0.5)))
    with pytest.raises(DomainError):
        mi_all_pairs_devices(mat, [])
    with pytest.raises((DomainError, NativeError)):
        mi_all_pairs_devices(mat, [0, 99])
