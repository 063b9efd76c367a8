"""Multi-GPU dispatcher: one process per GPU, upper-triangle tiles dealt across ranks.

The output tiles (I <= J) of the MI matrix are independent and all cost the
same (K = N), so the path shards with no data-path reduction
(SURVEY 8(e)): rank 0 holds the packed words; ONE broadcast sends them to
every rank (NCCL over NVLink, bit-packed so it is 1/8 of the int8 operand);
each rank unpacks the column blocks its tiles touch (``mi_rank_blocks``: half
of them at 8 ranks, whose tiles are dealt as column-group pairs) and computes
the tiles the C ABI's ``mi_tile_list(m, rank, world)`` deals it, writing each
tile and its mirror into its local output.  The MI matrix stays sharded; ``gather_to_root``
assembles it on request.

Everything here is plain torch.distributed plumbing around two callables,
so the same code runs over NCCL on GPUs and over gloo on CPU in the tests
(where the per-tile compute is supplied by the test).
"""

from __future__ import annotations

from typing import Callable

import numpy as np
import torch
import torch.distributed as dist

from . import _native as nat
from .binmat import n_words


def world_info(group=None) -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def rank_tiles(n_cols: int, rank: int, world: int) -> np.ndarray:
    """(k, 2) int32 (I, J) tiles of `rank`; the union over ranks is every I <= J
    tile exactly once (host logic in the C ABI, no device needed)."""
    return nat.tile_list(n_cols, rank, world)


def tile_mask(n_cols: int, tiles: np.ndarray, tile: int | None = None) -> np.ndarray:
    """Boolean m x m mask of the elements a tile list writes (tiles + mirrors)."""
    tile = tile or int(nat.lib().mi_tile_size())
    mask = np.zeros((n_cols, n_cols), dtype=bool)
    for I, J in np.asarray(tiles):
        r = slice(I * tile, min((I + 1) * tile, n_cols))
        c = slice(J * tile, min((J + 1) * tile, n_cols))
        mask[r, c] = True
        mask[c, r] = True
    return mask


def broadcast_words(words: torch.Tensor | None, n_rows: int, n_cols: int, device: torch.device,
                    src: int = 0, group=None) -> torch.Tensor:
    """The path's only collective: the packed words from `src` to every rank."""
    rank, _ = world_info(group)
    if rank == src:
        if words is None:
            raise ValueError("the source rank must provide the words")
        buf = words.to(device)
    else:
        buf = torch.empty((n_cols, n_words(n_rows)), dtype=torch.int64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.broadcast(buf, src=src, group=group)
    return buf


def run_sharded(words: torch.Tensor | None, n_rows: int, n_cols: int,
                compute: Callable[[torch.Tensor, np.ndarray, torch.Tensor], None],
                out: torch.Tensor, device: torch.device, group=None) -> np.ndarray:
    """Broadcast words, then compute this rank's tiles into `out`.

    ``compute(words_local, tiles, out)`` writes the given tiles and their
    mirrors into out.  Returns this rank's tile list.
    """
    rank, world = world_info(group)
    w = broadcast_words(words, n_rows, n_cols, device, group=group)
    tiles = rank_tiles(n_cols, rank, world)
    compute(w, tiles, out)
    return tiles


def stage_bounds(n_cols: int, stages: int) -> list[tuple[int, int, int, int]]:
    """Column groups of the staged broadcast: (first block, end block, first
    column, end column) per group, blocks of mi_tile_size() columns split as
    evenly as possible (the C ABI's staged host path cuts them the same way)."""
    tile = int(nat.lib().mi_tile_size())
    T = -(-n_cols // tile)
    S = max(1, min(stages, T))
    out = []
    for g in range(S):
        b0, b1 = T * g // S, T * (g + 1) // S
        out.append((b0, b1, min(b0 * tile, n_cols), min(b1 * tile, n_cols)))
    return out


def auto_stages(n_cols: int, world: int, num_sms: int) -> int:
    """Column groups for the staged broadcast: one per 8 tile rounds of a
    rank's share, at most 4, and none at world 1 (nothing to overlap).  Each
    extra group costs a partial tile round: measured at world 1
    (tools/stage_overhead.py) +0.58 ms on config 4 (26.0 ms) but +0.43 ms on
    config 3 (1.8 ms), so short shares stay in one piece."""
    if world <= 1:
        return 1
    tile = int(nat.lib().mi_tile_size())
    T = -(-n_cols // tile)
    rounds = T * (T + 1) // 2 / world / max(1, num_sms // 2)
    return int(max(1, min(4, rounds // 8)))


def run_sharded_staged(words: torch.Tensor | None, n_rows: int, n_cols: int,
                       begin: Callable[[], object],
                       stage: Callable[[object, torch.Tensor, int, int, int, np.ndarray, torch.Tensor], None],
                       out: torch.Tensor, device: torch.device, group=None, stages: int = 4,
                       src: int = 0) -> np.ndarray:
    """run_sharded with the broadcast cut into column groups that overlap the
    compute: every group's words go out as their own asynchronous broadcast,
    and once group g has arrived, ``stage(state, words, g, b0, b1, tiles_g,
    out)`` runs this rank's tiles whose larger block J lies in [b0, b1) (all
    their operands are then present).  ``begin()`` runs first and returns the
    state handed to every stage call.  Returns this rank's tile list."""
    rank, world = world_info(group)
    if rank == src:
        if words is None:
            raise ValueError("the source rank must provide the words")
        buf = words.to(device)
    else:
        buf = torch.empty((n_cols, n_words(n_rows)), dtype=torch.int64, device=device)
    bounds = stage_bounds(n_cols, stages)
    dist_on = dist.is_available() and dist.is_initialized()
    works = [dist.broadcast(buf[c0:c1], src=src, group=group, async_op=True) if dist_on and c1 > c0 else None
             for (_, _, c0, c1) in bounds]
    tiles = rank_tiles(n_cols, rank, world)
    state = begin()
    for g, (b0, b1, c0, c1) in enumerate(bounds):
        if works[g] is not None:
            works[g].wait()
        sel = tiles[(tiles[:, 1] >= b0) & (tiles[:, 1] < b1)] if len(tiles) else tiles
        stage(state, buf, g, b0, b1, sel, out)
    return tiles


def gather_to_root(out: torch.Tensor, n_cols: int, root: int = 0, group=None) -> torch.Tensor | None:
    """Assemble the full matrix on `root` from every rank's shard.

    ``out`` must be zero outside this rank's tiles and mirrors (allocate it
    with ``zero_fill=True``).  Every element is written by exactly one rank, so
    the sum-reduce onto the root is an exact gather (x + 0 == x in IEEE
    arithmetic).
    """
    rank, world = world_info(group)
    if world == 1:
        return out
    shard = out[:n_cols, :n_cols]
    if not shard.is_contiguous():
        shard = shard.contiguous()
    dist.reduce(shard, dst=root, op=dist.ReduceOp.SUM, group=group)
    return shard if rank == root else None


def mi_all_pairs_sharded(engine, words: torch.Tensor | None, n_rows: int, n_cols: int, cfg=None,
                         out_dtype: torch.dtype = torch.float64, out: torch.Tensor | None = None,
                         group=None, zero_fill: bool = False, stages: int | None = None
                         ) -> tuple[torch.Tensor, np.ndarray]:
    """GPU version: broadcast + unpack + fused Gram/MI over this rank's tiles.

    Returns (local output with this rank's tiles and mirrors written, tiles).
    ``zero_fill`` zeroes the rest of the local output, as gather_to_root needs.
    ``stages`` > 1: the broadcast goes out in that many column groups, each
    unpacked and its tiles computed as soon as it arrives
    (run_sharded_staged); the result is bit-identical.  None: auto_stages().
    """
    rank, world = world_info(group)
    if stages is None:
        stages = auto_stages(n_cols, world, engine.num_sms)
    if out is None:
        out = (torch.zeros if zero_fill else torch.empty)((n_cols, n_cols), dtype=out_dtype, device=engine.device)
    elif zero_fill:
        out.zero_()

    if stages > 1:
        tile = int(nat.lib().mi_tile_size())

        def begin():
            return engine.prepare_begin(n_rows, n_cols)

        def stage(prep, w, g, b0, b1, tiles_g, o):
            last = b1 * tile >= n_cols
            engine.prepare_range(prep, w, b0 * tile, prep.m_pad if last else b1 * tile, rank, world)
            if len(tiles_g):
                t = torch.from_numpy(np.ascontiguousarray(tiles_g, dtype=np.int32)).to(engine.device)
                engine.compute(prep, cfg, out_dtype, tiles=t, out=o)

        tiles = run_sharded_staged(words, n_rows, n_cols, begin, stage, out, engine.device, group, stages)
        return out, tiles

    def compute(w, tiles, o):
        prep = engine.prepare(w, n_rows, n_cols, rank, world)  # only this rank's column blocks
        engine.compute(prep, cfg, out_dtype, tiles=engine.tiles(n_cols, rank, world), out=o)

    tiles = run_sharded(words, n_rows, n_cols, compute, out, engine.device, group)
    return out, tiles


def copy_share_to_host(engine, local: torch.Tensor, n_cols: int, tiles: np.ndarray, host) -> None:
    """This rank's tiles and mirrors, device -> the shared host matrix
    (hostshm.SharedHostMatrix), as merged 2-D copies; returns once copied."""
    t = np.ascontiguousarray(np.asarray(tiles, dtype=np.int32))
    stream = torch.cuda.current_stream(engine.device)
    nat.check(nat.lib().mi_copy_tiles_to_host(local.data_ptr(), local.stride(0), n_cols, local.element_size(),
                                              t.ctypes.data, t.shape[0], host.ptr, n_cols, stream.cuda_stream),
              "mi_copy_tiles_to_host")
    stream.synchronize()


def mi_all_pairs_to_host(engine, words: torch.Tensor | None, n_rows: int, n_cols: int, host, cfg=None,
                         out_dtype: torch.dtype = torch.float64, out: torch.Tensor | None = None,
                         group=None, stages: int | None = None) -> np.ndarray:
    """Sharded compute, then every rank writes its share into the shared host
    matrix over its own PCIe link; after the barrier the full matrix is in
    ``host.array`` on every rank of the node."""
    local, tiles = mi_all_pairs_sharded(engine, words, n_rows, n_cols, cfg, out_dtype, out=out, group=group,
                                        stages=stages)
    copy_share_to_host(engine, local, n_cols, tiles, host)
    if dist.is_available() and dist.is_initialized():
        dist.barrier(group=group)
    return host.array

