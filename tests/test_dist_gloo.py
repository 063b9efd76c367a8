"""Multi-rank path on CPU: world_size 2 over gloo (127.0.0.1).

Exercises the dispatcher's host logic exactly as the NCCL run does: rank 0
holds the packed words, one broadcast sends them to every rank, each rank
computes only the upper-triangle tiles mi_tile_list() deals it (here with the
oracle standing in for the CUDA kernel -- test side only), and
gather_to_root() assembles the full matrix on rank 0, which must equal the
single-process oracle result bit for bit.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_stage(n_rows, n_cols, buf):
    """The per-stage compute the GPU path runs, with the C oracle standing in
    for the kernel (test side only): tile k of the stage into shard slot
    slot0 + k, tile-major like MI_TILE_MAJOR."""
    from oracle import oracle as O
    from paper_2411_19702_b200 import _native as nat

    tile = nat.lib().mi_tile_size()

    def stage(state, w, g, b0, b1, tiles_g, slot0):
        words = w.numpy().view(np.uint64)
        full = O.c_mi_all_pairs(words, n_rows)  # reference values, then keep only our tiles
        b = buf.numpy()
        for k, (I, J) in enumerate(np.asarray(tiles_g)):
            r0, c0 = I * tile, J * tile
            h, wd = min(tile, n_cols - r0), min(tile, n_cols - c0)
            b[slot0 + k, :h, :wd] = full[r0:r0 + h, c0:c0 + wd]

    return stage


def _worker(rank, world, port, n, m, result_q, stages=1):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2411_19702_b200 import _native as nat
        from paper_2411_19702_b200 import dispatch

        def ref_words():
            rng = np.random.default_rng(11)
            bits = (rng.random((n, m)) < 0.4).astype(np.uint8)
            return torch.from_numpy(O.pack_bits(bits).view(np.int64))

        words = ref_words() if rank == 0 else None
        tile = nat.lib().mi_tile_size()
        k = len(dispatch.rank_tiles(m, rank, world))
        buf = torch.zeros((max(k, 1), tile, tile), dtype=torch.float64)
        compute = _oracle_stage(n, m, buf)
        seen = []

        def stage(state, w, g, b0, b1, tiles_g, slot0):
            # the tiles of this group touch only columns that have arrived:
            # columns [0, c1) must already hold the source's words
            c1 = dispatch.stage_bounds(m, stages)[g][3]
            assert torch.equal(w[:c1], ref_words()[:c1])
            seen.append(len(tiles_g))
            compute(state, w, g, b0, b1, tiles_g, slot0)

        tiles = dispatch.run_sharded(words, n, m, lambda: None, stage, torch.device("cpu"), stages=stages)
        assert sum(seen) == len(tiles) == k
        shard = dispatch.Shard(m, tile, tiles, buf[:len(tiles)])
        # the shard holds ~1/world of the triangle, not an m x m matrix
        assert shard.nbytes <= max(k, 1) * tile * tile * 8
        full = dispatch.gather_to_root(shard)
        if rank == 0:
            ref = O.c_mi_all_pairs(words.numpy().view(np.uint64), n)
            result_q.put(("ok", bool(np.array_equal(full.numpy(), ref)), len(tiles)))
        else:
            assert full is None
            result_q.put(("peer", True, len(tiles)))
    except Exception as exc:  # pragma: no cover - surfaced through the queue
        import traceback
        result_q.put(("error", repr(exc) + traceback.format_exc(), 0))
    finally:
        dist.destroy_process_group()


def _run(world, n, m, stages):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, m, q, stages)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    errors = [r for r in results if r[0] == "error"]
    assert not errors, errors
    root = [r for r in results if r[0] == "ok"][0]
    assert root[1], "gathered matrix differs from the single-process oracle"
    return results


@pytest.mark.parametrize("stages", [1, 2, 3])
@pytest.mark.parametrize("n,m", [(300, 600), (1000, 300), (200, 1100)])
def test_two_rank_broadcast_shard_gather(n, m, stages):
    """One broadcast (stages 1) or column-group broadcasts overlapping the
    per-group compute (dispatch.run_sharded): tile-major shards, gathered to
    rank 0 point to point (no reduction), equal the single-process oracle."""
    results = _run(2, n, m, stages)
    # both ranks got work when there is more than one tile
    assert all(r[2] >= 1 for r in results) or m <= 256


@pytest.mark.parametrize("stages", [1, 2])
def test_four_rank_column_group_shares(stages):
    """4 ranks (T >= 16 tile columns: each rank holds 3 of 4 column groups),
    gathered bit-identically."""
    results = _run(4, 200, 16 * 256 + 37, stages)
    counts = sorted(r[2] for r in results)
    assert counts[-1] - counts[0] <= 4


def test_four_rank_dealing_holds_three_quarters():
    """The 4-rank deal: every tile once, shares within a few tiles, and each
    rank's blocks (what it unpacks) 3/4 of X."""
    from paper_2411_19702_b200 import _native as nat

    for m in (16 * 256, 50_000, 20_000):
        T = -(-m // 256)
        shares = [nat.tile_list(m, r, 4) for r in range(4)]
        allt = np.concatenate(shares)
        assert len(allt) == T * (T + 1) // 2 and len({tuple(x) for x in allt}) == len(allt)
        sizes = [len(x) for x in shares]
        assert max(sizes) - min(sizes) <= max(4, T // 8)
        for r in range(4):
            used = int(nat.rank_blocks(m, r, 4).sum())
            assert used <= -(-3 * T // 4) + 1
