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


def _oracle_compute(n_rows, n_cols):
    from oracle import oracle as O
    from paper_2411_19702_b200 import _native as nat

    tile = nat.lib().mi_tile_size()

    def compute(w, tiles, out):
        words = w.numpy().view(np.uint64)
        full = O.c_mi_all_pairs(words, n_rows)  # reference values, then keep only our tiles
        o = out.numpy()
        for I, J in np.asarray(tiles):
            r = slice(I * tile, min((I + 1) * tile, n_cols))
            c = slice(J * tile, min((J + 1) * tile, n_cols))
            o[r, c] = full[r, c]
            o[c, r] = full[c, r]

    return compute


def _worker(rank, world, port, n, m, result_q, stages=1):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2411_19702_b200 import dispatch

        words = None
        if rank == 0:
            rng = np.random.default_rng(11)
            bits = (rng.random((n, m)) < 0.4).astype(np.uint8)
            words = torch.from_numpy(O.pack_bits(bits).view(np.int64))
        out = torch.zeros((m, m), dtype=torch.float64)
        if stages == 1:
            tiles = dispatch.run_sharded(words, n, m, _oracle_compute(n, m), out, torch.device("cpu"))
        else:
            compute = _oracle_compute(n, m)
            seen = []

            def stage(state, w, g, b0, b1, tiles_g, o):
                # the tiles of this group touch only columns that have arrived:
                # columns [0, c1) must already hold the source's words
                c1 = dispatch.stage_bounds(m, stages)[g][3]
                ref_w = torch.from_numpy(O.pack_bits((np.random.default_rng(11).random((n, m)) < 0.4)
                                                     .astype(np.uint8)).view(np.int64))
                assert torch.equal(w[:c1], ref_w[:c1])
                seen.append(len(tiles_g))
                compute(w, tiles_g, o)

            tiles = dispatch.run_sharded_staged(words, n, m, lambda: None, stage, out, torch.device("cpu"),
                                                stages=stages)
            assert sum(seen) == len(tiles)
        full = dispatch.gather_to_root(out, m)
        if rank == 0:
            ref = O.c_mi_all_pairs(words.numpy().view(np.uint64), n)
            result_q.put(("ok", bool(np.array_equal(full.numpy(), ref)), len(tiles)))
        else:
            result_q.put(("peer", True, len(tiles)))
    except Exception as exc:  # pragma: no cover - surfaced through the queue
        result_q.put(("error", repr(exc), 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("stages", [1, 2, 3])
@pytest.mark.parametrize("n,m", [(300, 600), (1000, 300), (200, 1100)])
def test_two_rank_broadcast_shard_gather(n, m, stages):
    """One broadcast (stages 1) or column-group broadcasts overlapping the
    per-group compute (dispatch.run_sharded_staged): the same gathered matrix."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, m, q, stages)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    errors = [r for r in results if r[0] == "error"]
    assert not errors, errors
    root = [r for r in results if r[0] == "ok"][0]
    assert root[1], "gathered matrix differs from the single-process oracle"
    # both ranks got work when there is more than one tile
    assert all(r[2] >= 1 for r in results) or m <= 256
