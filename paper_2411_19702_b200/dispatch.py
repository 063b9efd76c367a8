"""Multi-GPU dispatcher: one process per GPU, upper-triangle tiles dealt across ranks.

The output tiles (I <= J) of the MI matrix are independent and all cost the
same (K = N), so the path shards with no data-path reduction (
the reference computes the same triangle in one process,
/root/reference/pkg/src/mimatrix/_kernels.py:53-61, and mirrors it,
engine.py:137-138): rank 0 holds the packed words; ONE broadcast sends them
to every rank (NCCL over NVLink, bit-packed: 1/4 of the e2m1 operand); each
rank unpacks only the column blocks its tiles touch (``mi_rank_blocks``: 3/4
of them at 4 ranks, 1/2 at 8) and computes the tiles ``mi_tile_list(m, rank,
world)`` deals it.

The result stays sharded: a ``Shard`` holds this rank's tiles tile-major
(tile k of its list in slot k, TS x TS, no mirrors -- MI_TILE_MAJOR), i.e.
~m^2 / (2 world) elements per rank instead of an m x m matrix.  Gathering is
on request and is never a reduction:

* ``gather_to_root``: point-to-point sends of the shards to the root, which
  places tiles and mirrors into its m x m matrix (``mi_scatter_tiles``);
* ``mi_all_pairs_to_host``: every rank writes its own tiles and mirrors
  straight into one pinned host matrix shared by the node's ranks
  (``hostshm.SharedHostMatrix``), over its own PCIe link (zero-copy kernel).

The broadcast can be staged (``stages`` > 1): one asynchronous broadcast per
column group, each group unpacked and its tiles computed as soon as it lands.

Everything except the two GPU entry points is plain torch.distributed
plumbing around callables, so the same code runs over NCCL on GPUs and over
gloo on CPU in the tests (where the per-tile compute is supplied by the test).
"""

from __future__ import annotations

from dataclasses import dataclass
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
    """Boolean m x m mask of the elements a tile list covers (tiles + mirrors)."""
    tile = tile or int(nat.lib().mi_tile_size())
    mask = np.zeros((n_cols, n_cols), dtype=bool)
    for I, J in np.asarray(tiles):
        r = slice(I * tile, min((I + 1) * tile, n_cols))
        c = slice(J * tile, min((J + 1) * tile, n_cols))
        mask[r, c] = True
        mask[c, r] = True
    return mask


@dataclass
class Shard:
    """One rank's part of the MI matrix: tile k of ``tiles`` ((I, J), I <= J)
    is ``buf[k]`` (TS x TS, row i - I TS, column j - J TS; rows / columns past
    m are not written).  Mirrors are implied (MI is symmetric)."""

    n_cols: int
    tile: int
    tiles: np.ndarray      # (k, 2) int32, slot order
    buf: torch.Tensor      # (k, TS, TS)

    @property
    def nbytes(self) -> int:
        return self.buf.numel() * self.buf.element_size()

    def tiles_device(self) -> torch.Tensor:
        return torch.from_numpy(np.ascontiguousarray(self.tiles, dtype=np.int32)).to(self.buf.device)

    def place(self, out, mirror: bool = True) -> None:
        """Write these tiles (and their mirrors) into the full matrix ``out``:
        a device tensor, or a pinned (mi_host_register'ed) host array, which
        the device writes over PCIe.  CPU shards (the gloo tests) are placed
        with plain slicing."""
        if self.buf.device.type == "cpu":
            o = out if isinstance(out, np.ndarray) else out.numpy()
            b = self.buf.numpy()
            m, ts = self.n_cols, self.tile
            for k, (I, J) in enumerate(np.asarray(self.tiles)):
                r0, c0 = I * ts, J * ts
                h, w = min(ts, m - r0), min(ts, m - c0)
                o[r0:r0 + h, c0:c0 + w] = b[k, :h, :w]
                if mirror and I != J:
                    o[c0:c0 + w, r0:r0 + h] = b[k, :h, :w].T
            return
        if len(self.tiles) == 0:
            return
        if isinstance(out, np.ndarray):
            ptr, ld, esz = out.ctypes.data, out.strides[0] // out.itemsize, out.itemsize
        else:
            ptr, ld, esz = out.data_ptr(), out.stride(0), out.element_size()
        if esz != self.buf.element_size():
            raise ValueError("out dtype differs from the shard's")
        t = self.tiles_device()
        stream = torch.cuda.current_stream(self.buf.device)
        nat.check(nat.lib().mi_scatter_tiles(self.buf.data_ptr(), t.data_ptr(), len(self.tiles), self.n_cols, esz,
                                             ptr, ld, 1 if mirror else 0, stream.cuda_stream),
                  "mi_scatter_tiles")
        stream.synchronize()  # t and the destination must outlive the kernel


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


def stage_order(tiles: np.ndarray, bounds) -> tuple[np.ndarray, list[tuple[int, int]]]:
    """The rank's tiles reordered so that each stage's tiles (larger block J in
    the stage's block range) are contiguous, keeping the dealt (banded) order
    inside a stage; returns (tiles, [(first slot, end slot) per stage])."""
    tiles = np.asarray(tiles, dtype=np.int32).reshape(-1, 2)
    parts, spans, k = [], [], 0
    for b0, b1, _, _ in bounds:
        sel = tiles[(tiles[:, 1] >= b0) & (tiles[:, 1] < b1)]
        parts.append(sel)
        spans.append((k, k + len(sel)))
        k += len(sel)
    return (np.concatenate(parts) if parts else tiles), spans


def run_sharded(words: torch.Tensor | None, n_rows: int, n_cols: int,
                begin: Callable[[], object],
                stage: Callable[[object, torch.Tensor, int, int, int, np.ndarray, int], None],
                device: torch.device, group=None, stages: int = 1, src: int = 0) -> np.ndarray:
    """Broadcast the words (as ``stages`` asynchronous column-group broadcasts)
    and run this rank's tiles stage by stage: once group g has landed,
    ``stage(state, words, g, b0, b1, tiles_g, slot0)`` computes the rank's
    tiles whose larger block J lies in [b0, b1) (all their operands are then
    present) into shard slots slot0.. .  ``begin()`` runs first and returns
    the state handed to every stage call.  Returns the rank's tiles in slot
    order."""
    rank, world = world_info(group)
    if rank == src:
        if words is None:
            raise ValueError("the source rank must provide the words")
        buf = words.to(device)
    else:
        buf = torch.empty((n_cols, n_words(n_rows)), dtype=torch.int64, device=device)
    bounds = stage_bounds(n_cols, stages)
    dist_on = dist.is_available() and dist.is_initialized() and world > 1
    if dist_on and len(bounds) == 1:
        dist.broadcast(buf, src=src, group=group)
        works = [None]
    else:
        works = [dist.broadcast(buf[c0:c1], src=src, group=group, async_op=True) if dist_on and c1 > c0 else None
                 for (_, _, c0, c1) in bounds]
    tiles, spans = stage_order(rank_tiles(n_cols, rank, world), bounds)
    state = begin()
    for g, (b0, b1, c0, c1) in enumerate(bounds):
        if works[g] is not None:
            works[g].wait()
        s0, s1 = spans[g]
        stage(state, buf, g, b0, b1, tiles[s0:s1], s0)
    return tiles


def mi_all_pairs_sharded(engine, words: torch.Tensor | None, n_rows: int, n_cols: int, cfg=None,
                         out_dtype: torch.dtype = torch.float64, group=None, stages: int | None = None,
                         buf: torch.Tensor | None = None, timing: list | None = None) -> Shard:
    """GPU path: broadcast + unpack of this rank's column blocks + fused
    Gram/MI over this rank's tiles, stored tile-major (MI_TILE_MAJOR).
    ``stages`` > 1: the broadcast goes out in that many column groups, each
    unpacked and its tiles computed as soon as it arrives; None: auto_stages().
    ``buf``: a reusable (>= k, TS, TS) output.  ``timing``: if a list, a pair
    of CUDA events recorded around each fused-kernel launch is appended (the
    bench's roofline).  The values are bit-identical to the one-GPU matrix at
    the same positions."""
    rank, world = world_info(group)
    if stages is None:
        stages = auto_stages(n_cols, world, engine.num_sms)
    stages = max(1, int(stages))
    tile = int(nat.lib().mi_tile_size())
    k = len(rank_tiles(n_cols, rank, world))
    if buf is None or buf.shape[0] < k or buf.dtype != out_dtype:
        buf = torch.empty((max(k, 1), tile, tile), dtype=out_dtype, device=engine.device)

    def fused(prep, t, out):
        if timing is None:
            engine.compute(prep, cfg, out_dtype, tiles=t, out=out, tile_major=True)
            return
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream = torch.cuda.current_stream(engine.device)
        e0.record(stream)
        engine.compute(prep, cfg, out_dtype, tiles=t, out=out, tile_major=True)
        e1.record(stream)
        timing.append((e0, e1))

    def begin():
        return engine.prepare_begin(n_rows, n_cols)

    # device copies of the per-stage tile lists, cached on the engine (a
    # pageable H2D per step would stall the host behind the stream)
    key = ("stage_tiles", n_cols, rank, world, stages, nat.get_tuning("cta_group"), nat.get_tuning("band"),
           nat.get_tuning("shard"))
    cache = engine._tiles.get(key)
    if cache is None:
        order, spans = stage_order(rank_tiles(n_cols, rank, world), stage_bounds(n_cols, stages))
        cache = {s0: torch.from_numpy(np.ascontiguousarray(order[s0:s1])).to(engine.device)
                 for s0, s1 in spans if s1 > s0}
        engine._tiles[key] = cache

    def stage(prep, w, g, b0, b1, tiles_g, slot0):
        last = b1 * tile >= n_cols
        engine.prepare_range(prep, w, b0 * tile, prep.m_pad if last else b1 * tile, rank, world)
        if len(tiles_g):
            fused(prep, cache[slot0], buf[slot0:slot0 + len(tiles_g)])

    if stages <= 1:
        def begin1():
            return None

        def stage1(_, w, g, b0, b1, tiles_g, slot0):
            prep = engine.prepare(w, n_rows, n_cols, rank, world)  # only this rank's column blocks
            if len(tiles_g):
                fused(prep, cache[slot0], buf[slot0:slot0 + len(tiles_g)])

        tiles = run_sharded(words, n_rows, n_cols, begin1, stage1, engine.device, group, 1)
    else:
        tiles = run_sharded(words, n_rows, n_cols, begin, stage, engine.device, group, stages)
    return Shard(n_cols, tile, tiles, buf[:len(tiles)])


def gather_to_root(shard: Shard, root: int = 0, group=None, out: torch.Tensor | None = None):
    """Assemble the full m x m matrix on `root` from every rank's shard: each
    rank sends its tile list and tile-major buffer point to point; the root
    places every shard's tiles and mirrors (mi_scatter_tiles).  No reduction:
    each element is written exactly once.  Returns the matrix on the root,
    None elsewhere."""
    rank, world = world_info(group)
    m = shard.n_cols
    dev = shard.buf.device
    # NCCL moves device tensors; gloo point-to-point takes host tensors
    wire = dev if (world > 1 and dist.get_backend(group) == "nccl") else torch.device("cpu")
    if rank == root:
        if out is None:
            out = torch.empty((m, m), dtype=shard.buf.dtype, device=dev)
        shard.place(out)
        if world == 1:
            return out
        for r in range(world):
            if r == root:
                continue
            k = torch.zeros((1,), dtype=torch.int64, device=wire)
            dist.recv(k, src=r, group=group)
            n = int(k.item())
            if n == 0:
                continue
            tl = torch.empty((n, 2), dtype=torch.int32, device=wire)
            dist.recv(tl, src=r, group=group)
            b = torch.empty((n, shard.tile, shard.tile), dtype=shard.buf.dtype, device=wire)
            dist.recv(b, src=r, group=group)
            Shard(m, shard.tile, tl.cpu().numpy(), b.to(dev)).place(out)
        return out
    n = len(shard.tiles)
    dist.send(torch.tensor([n], dtype=torch.int64, device=wire), dst=root, group=group)
    if n:
        dist.send(torch.from_numpy(np.ascontiguousarray(shard.tiles, dtype=np.int32)).to(wire), dst=root, group=group)
        dist.send(shard.buf.contiguous().to(wire), dst=root, group=group)
    return None


def mi_all_pairs_to_host(engine, words: torch.Tensor | None, n_rows: int, n_cols: int, host, cfg=None,
                         out_dtype: torch.dtype = torch.float64, group=None, stages: int | None = None,
                         buf: torch.Tensor | None = None) -> np.ndarray:
    """Sharded compute, then every rank writes its tiles and mirrors straight
    into the shared pinned host matrix (``host.array``, mapped) over its own
    PCIe link; after the barrier the full matrix is there on every rank of the
    node."""
    shard = mi_all_pairs_sharded(engine, words, n_rows, n_cols, cfg, out_dtype, group=group, stages=stages, buf=buf)
    shard.place(host.array)
    if dist.is_available() and dist.is_initialized():
        dist.barrier(group=group)
    return host.array
