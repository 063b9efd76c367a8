"""Multi-rank GPU path: 2-4 ranks on the one visible GPU, collectives over gloo.

The round's GPU box exposes a single B200, so this runs the exact NCCL-run
code path (broadcast of the packed words from rank 0, per-rank tile lists from
mi_tile_list, partial unpacks of the rank's column blocks, the fused kernel on
only those tiles into a tile-major shard, point-to-point sends of the shards
to rank 0, which places tiles and mirrors with mi_scatter_tiles) with gloo
carrying the host-staged collectives.  The kernels of the ranks never wait on
each other.  The gathered matrix must equal the single-process result bit for
bit.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, m, cfg_id, dtype_name, result_q, stages=1):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_19702_b200 import dispatch
        from paper_2411_19702_b200 import datagen
        from paper_2411_19702_b200.engine import EngineConfig, MIEngine

        torch.cuda.set_device(0)
        eng = MIEngine.get(0)
        dtype = getattr(torch, dtype_name)
        words = datagen.generate_words_device(datagen.config_recipe(cfg_id, n, m), eng.device) if rank == 0 else None
        cfg = EngineConfig()
        shard = dispatch.mi_all_pairs_sharded(eng, words, n, m, cfg, dtype, stages=stages)
        tiles = shard.tiles
        # the shard holds only this rank's tiles: ~1/world of the triangle
        assert shard.buf.shape[0] == len(tiles) or len(tiles) == 0
        full = dispatch.gather_to_root(shard)
        torch.cuda.synchronize()
        if rank == 0:
            prep = eng.prepare(words, n, m)
            ref = eng.compute(prep, cfg, dtype)
            torch.cuda.synchronize()
            same = bool(torch.equal(full, ref[:m, :m]))
            result_q.put(("ok", same, len(tiles)))
        else:
            result_q.put(("peer", True, len(tiles)))
    except Exception as exc:  # pragma: no cover - surfaced through the queue
        import traceback
        result_q.put(("error", repr(exc) + traceback.format_exc(), 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("stages", [1, 4])
@pytest.mark.parametrize("world,n,m,cfg_id,dtype", [
    (2, 10_000, 2_000, 2, "float64"),
    (2, 4_097, 1_300, 4, "float32"),
    (2, 1_000, 257, 1, "float64"),
    (4, 3_000, 4_400, 4, "float32"),
    (4, 2_000, 4_200, 2, "float64"),
])
def test_multi_rank_sharded_gather_matches_single(world, n, m, cfg_id, dtype, stages):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, m, cfg_id, dtype, q, stages))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    errors = [r for r in results if r[0] == "error"]
    assert not errors, errors
    root = [r for r in results if r[0] == "ok"][0]
    assert root[1], "gathered matrix differs from the single-process result"
    assert sum(r[2] for r in results) >= 1


@pytest.mark.parametrize("world", [4, 8])
@pytest.mark.parametrize("n,m,dtype", [(20_000, 4_300, "float64"), (6_000, 4_100, "float32")])
def test_group_dealt_shares_in_one_process(engine, world, n, m, dtype):
    """The 4- and 8-rank column-group dealing with per-rank partial unpacks
    (mi_rank_blocks + mi_unpack_colsum_blocks), run rank by rank in one
    process into tile-major shards (MI_TILE_MAJOR) and placed with
    mi_scatter_tiles: together exactly the 1-rank matrix."""
    import numpy as np
    from oracle import oracle as O
    from paper_2411_19702_b200 import _native as nat
    from paper_2411_19702_b200 import dispatch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    dt = getattr(torch, dtype)
    rng = np.random.default_rng(m)
    words = O.pack_bits((rng.random((n, m)) < 0.35).astype(np.uint8))
    dev = engine.upload(words)
    full = engine.all_pairs_device(dev, n, m, None, dt)
    acc = torch.full_like(full, float("nan"))
    T = -(-m // nat.lib().mi_tile_size())
    for r in range(world):
        frac = {4: 3 * T // 4, 8: T // 2}[world]
        assert int(nat.rank_blocks(m, r, world).sum()) <= frac + 2
        prep = engine.prepare(dev, n, m, r, world)
        t = engine.tiles(m, r, world)
        buf = engine.compute(prep, None, dt, tiles=t, tile_major=True)
        dispatch.Shard(m, nat.lib().mi_tile_size(), t.cpu().numpy(), buf[:t.shape[0]]).place(acc)
    torch.cuda.synchronize()
    assert torch.equal(acc, full)


def test_scatter_into_pinned_host_matrix(engine):
    """mi_scatter_tiles straight into registered host memory (zero-copy over
    PCIe) equals the device matrix; pageable destinations are refused."""
    import numpy as np
    from oracle import oracle as O
    from paper_2411_19702_b200 import _native as nat
    from paper_2411_19702_b200 import dispatch
    from paper_2411_19702_b200.errors import DomainError

    n, m = 3_000, 1_500
    rng = np.random.default_rng(5)
    dev = engine.upload(O.pack_bits((rng.random((n, m)) < 0.3).astype(np.uint8)))
    full = engine.all_pairs_device(dev, n, m).cpu().numpy()
    prep = engine.prepare(dev, n, m)
    t = engine.tiles(m)
    shard = dispatch.Shard(m, nat.lib().mi_tile_size(), t.cpu().numpy(),
                           engine.compute(prep, None, torch.float64, tiles=t, tile_major=True))
    host = np.full((m, m), np.nan)
    with pytest.raises(DomainError):
        shard.place(host)  # pageable: not writable by the device
    nat.check(nat.lib().mi_host_register(host.ctypes.data, host.nbytes))
    try:
        shard.place(host)
    finally:
        nat.lib().mi_host_unregister(host.ctypes.data)
    assert np.array_equal(host, full)


def _host_worker(rank, world, port, n, m, name, result_q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    host = None
    try:
        from paper_2411_19702_b200 import datagen, dispatch
        from paper_2411_19702_b200.engine import MIEngine
        from paper_2411_19702_b200.hostshm import SharedHostMatrix

        torch.cuda.set_device(0)
        eng = MIEngine.get(0)
        if rank == 0:
            host = SharedHostMatrix(name, m, np.float64, create=True)
        dist.barrier()
        if rank != 0:
            host = SharedHostMatrix(name, m, np.float64, create=False)
        words = datagen.generate_words_device(datagen.config_recipe(2, n, m), eng.device) if rank == 0 else None
        full = dispatch.mi_all_pairs_to_host(eng, words, n, m, host)
        if rank == 0:
            ref = eng.all_pairs_device(words, n, m).cpu().numpy()
            result_q.put(("ok", bool(np.array_equal(full, ref)), 0))
        else:
            result_q.put(("peer", True, 0))
        dist.barrier()
    except Exception as exc:  # pragma: no cover
        import traceback
        result_q.put(("error", repr(exc) + traceback.format_exc(), 0))
    finally:
        if host is not None:
            host.close()
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ranks_write_one_shared_host_matrix(world):
    """Every rank writes its tiles and mirrors into one POSIX shared-memory
    host matrix (mi_host_register + mi_scatter_tiles, zero-copy); the
    assembled matrix equals the single-process result."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    name = f"mi_b200_test_{os.getpid()}_{world}"
    procs = [ctx.Process(target=_host_worker, args=(r, world, port, 5_000, 1_300, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    errors = [r for r in results if r[0] == "error"]
    assert not errors, errors
    assert [r for r in results if r[0] == "ok"][0][1]
