"""All-pairs binary mutual information on B200 -- the drop-in entry point.

``mi_all_pairs(data, cfg=None, backend="dense", threads=0) -> MIMatrix`` keeps
the reference's signature, defaults, output layout (fresh C-contiguous m x m
float64, bit-identical symmetric, diagonal = column entropy) and error
behaviour (engine.py:144-168 of /root/reference/pkg/src/mimatrix).  Its body
is: H2D of the packed words -> kernel 1 (unpack + column sums) -> kernel 2+3
(tcgen05 int8 Gram over upper-triangle tiles with the MI epilogue fused on the
TMEM accumulators) -> D2H.  All three backends of the reference run this one
GPU path (there is no CPU fallback and no multi-backend dispatch); the
backend name is still validated exactly like the reference does.

``MIEngine`` is the device API: device-resident inputs and outputs (torch
tensors, used only as device memory and streams), float32 or float64 output,
tile subsets for the multi-GPU dispatcher, and the int32 count export used for
bit-exact parity.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .binmat import as_dense_words, n_words
from .errors import DimensionError, DomainError, NativeError

MODES = ("exact", "epsilon")
BACKENDS = ("dense", "sparse", "direct")


@dataclass(frozen=True)
class EngineConfig:
    """Evaluation options for MI assembly (engine.py:32-44)."""

    mode: str = "exact"
    epsilon: float = 1e-12
    include_diagonal: bool = True

    def __post_init__(self):
        if self.mode not in MODES:
            raise DomainError(f"mode must be one of {MODES}, got {self.mode!r}")
        if not self.epsilon > 0:
            raise DomainError(f"epsilon must be positive, got {self.epsilon}")


@dataclass(frozen=True, eq=False)
class MIMatrix:
    """Symmetric m x m matrix of pairwise mutual information, in bits (engine.py:66-78)."""

    values: np.ndarray

    @property
    def n_cols(self) -> int:
        return self.values.shape[0]

    def checksum(self) -> float:
        return float(self.values.sum())


def _config_fields(cfg) -> tuple[int, float, int]:
    """Accept our EngineConfig or the reference's (same fields)."""
    if cfg is None:
        cfg = EngineConfig()
    mode = getattr(cfg, "mode", None)
    eps = getattr(cfg, "epsilon", None)
    if mode not in MODES:
        raise DomainError(f"mode must be one of {MODES}, got {mode!r}")
    if eps is None or not eps > 0:
        raise DomainError(f"epsilon must be positive, got {eps}")
    return MODES.index(mode), float(eps), int(bool(getattr(cfg, "include_diagonal", True)))


_OUT_KIND = {torch.float64: nat.MI_OUT_F64, torch.float32: nat.MI_OUT_F32, torch.int32: nat.MI_OUT_COUNTS}


@dataclass
class Prepared:
    """Device-resident operand of one dataset: K-major X (or, on the word-operand
    path, the packed words themselves) and column sums."""

    n_rows: int
    n_cols: int
    ld: int          # bytes per X row (N_pad)
    m_pad: int       # X rows
    x: torch.Tensor | None  # int8 (m_pad, ld); None on the word-operand path
    colsum: torch.Tensor  # int32 (m_pad,)
    colstat: torch.Tensor  # uint8 workspace (mi_colstat_bytes): marginals + their log2 splits
    perm: torch.Tensor | None = None  # order "colsum": int32 slot -> column (X, colsum, colstat in slot order)
    inv: torch.Tensor | None = None   # order "colsum": int32 column -> slot
    words: torch.Tensor | None = None  # word-operand path: the (m, nw) words the GEMM expands itself
    layout_knobs: tuple = ()  # ("fp4", "cta_group") at prepare time: X's format depends on them
    stats_ready: bool = True  # False: the word-operand path's first compute() also computes the statistics

    def __post_init__(self):
        if not self.layout_knobs:
            self.layout_knobs = _layout_knobs()


def _layout_knobs() -> tuple:
    """The knobs that fix the operand format (e2m1 or int8 X, tile size)."""
    return (nat.get_tuning("fp4"), nat.get_tuning("cta_group"))


ORDERS = ("natural", "colsum", "auto")
# measured steps (tools/order_probe.py): config 4 (m = 50,000) colsum 25.3 vs natural 25.9 ms,
# config 5 (m = 20,000) 64.5 vs 66.5 ms, config 2 (m = 2,000) 0.35 vs 0.11 ms
AUTO_ORDER_MIN_COLS = 16384


def _stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class MIEngine:
    """Per-device engine.  Allocation goes through torch's caching allocator;
    kernels are enqueued on torch's current stream of that device."""

    _instances: dict[int, "MIEngine"] = {}
    _lock = threading.Lock()

    def __init__(self, device: int | torch.device | None = None):
        if not torch.cuda.is_available():
            raise NativeError("no CUDA device visible: the MI engine runs only on B200 (sm_100a)")
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device if isinstance(device, int) else device.index or 0)
        self.num_sms, major, minor = nat.device_info(self.device.index)
        self._tiles: dict[tuple, torch.Tensor] = {}

    @classmethod
    def get(cls, device: int | torch.device | None = None) -> "MIEngine":
        if device is None:
            if not torch.cuda.is_available():
                raise NativeError("no CUDA device visible: the MI engine runs only on B200 (sm_100a)")
            device = torch.cuda.current_device()
        idx = device if isinstance(device, int) else (device.index or 0)
        with cls._lock:
            if idx not in cls._instances:
                cls._instances[idx] = cls(idx)
            return cls._instances[idx]

    # ------------------------------------------------------------------ layout
    @staticmethod
    def layout(n_rows: int, n_cols: int) -> tuple[int, int]:
        L = nat.lib()
        return int(L.mi_kmajor_ld(n_rows)), int(L.mi_kmajor_rows(n_cols))

    def tiles(self, n_cols: int, rank: int = 0, world: int = 1) -> torch.Tensor:
        # the list depends on the tile size (cta_group) and order (band) knobs
        key = (n_cols, rank, world, nat.get_tuning("cta_group"), nat.get_tuning("band"), nat.get_tuning("shard"))
        t = self._tiles.get(key)
        if t is None:
            host = nat.tile_list(n_cols, rank, world)
            t = torch.from_numpy(np.ascontiguousarray(host)).to(self.device)
            self._tiles[key] = t
        return t

    # ------------------------------------------------------------------ stages
    def pack_bits(self, bits_dev: torch.Tensor, check: bool = True) -> torch.Tensor:
        """binmat.from_bits / from_rows on the device (mi_pack_bits): a
        row-major (N, m) uint8 / bool 0/1 tensor -> words (m, nw) int64.  With
        ``check`` a non-binary byte raises DomainError like the reference's
        from_rows (one 4-byte read back)."""
        if bits_dev.device != self.device or bits_dev.dim() != 2 or bits_dev.element_size() != 1 \
                or bits_dev.dtype not in (torch.uint8, torch.bool, torch.int8):
            raise DimensionError("bits must be an (N, m) uint8/bool tensor on the engine's device")
        n, m = int(bits_dev.shape[0]), int(bits_dev.shape[1])
        if n < 1 or m < 1:
            raise DimensionError("matrix must have at least one row and one column")
        if bits_dev.stride(1) != 1 or (n > 1 and bits_dev.stride(0) < m):
            bits_dev = bits_dev.contiguous()  # the kernel reads rows with unit column stride
        ld = bits_dev.stride(0) if n > 1 else m
        words = torch.empty((m, n_words(n)), dtype=torch.int64, device=self.device)
        bad = torch.zeros((1,), dtype=torch.int32, device=self.device)
        nat.check(nat.lib().mi_pack_bits(bits_dev.data_ptr(), n, m, ld, words.data_ptr(),
                                         bad.data_ptr(), _stream_ptr(self.device)),
                  "mi_pack_bits")
        if check and int(bad.item()) != 0:
            raise DomainError("values must be 0 or 1")
        return words

    def from_bits(self, bits: np.ndarray):
        """binmat.from_bits / from_rows for a large host uint8 / bool 0/1
        matrix, packed on the GPU: H2D of the bytes, pack_bits, D2H of the
        words (1/8 of the bytes) -> BinaryMatrix.  1e5 x 1e4 (1 GB of
        pageable bytes): 147 ms against 2.6 s for numpy's packbits."""
        from .binmat import BinaryMatrix

        arr = np.asarray(bits)
        if arr.ndim != 2 or arr.shape[0] < 1 or arr.shape[1] < 1:
            raise DimensionError("expected a non-empty 2-d (N, m) matrix")
        if arr.dtype not in (np.uint8, np.bool_):
            if not np.issubdtype(arr.dtype, np.integer):
                raise DomainError(f"values must be integer 0/1, got dtype {arr.dtype}")
            if np.any((arr != 0) & (arr != 1)):
                raise DomainError("values must be 0 or 1")
            arr = arr.astype(np.uint8)
        host = torch.from_numpy(np.ascontiguousarray(arr).view(np.uint8))
        words = self.pack_bits(host.to(self.device, non_blocking=False))
        return BinaryMatrix(int(arr.shape[0]), int(arr.shape[1]), words.cpu().numpy().view(np.uint64))

    def from_sparse(self, sparse) -> torch.Tensor:
        """binmat.to_dense (binmat.py:187-194) on the device for the sparse
        backend's data (a SparseBinaryMatrix: per-column sorted row-index
        lists): upload the CSC index arrays, set the bits (mi_pack_sparse; cost
        ~ nnz, no N x m host matrix).  Returns device words (m, nw)."""
        n, m = int(sparse.n_rows), int(sparse.n_cols)
        if n < 1 or m < 1:
            raise DimensionError("matrix must have at least one row and one column")
        cols = [np.asarray(ix, dtype=np.int64).ravel() for ix in sparse.col_indices]
        if len(cols) != m:
            raise DimensionError("col_indices must hold one list per column")
        indptr = np.zeros(m + 1, dtype=np.int64)
        np.cumsum([c.size for c in cols], out=indptr[1:])
        idx = np.concatenate(cols) if indptr[-1] else np.zeros(1, dtype=np.int64)
        d_idx = torch.from_numpy(idx).to(self.device)
        d_ptr = torch.from_numpy(indptr).to(self.device)
        words = torch.empty((m, n_words(n)), dtype=torch.int64, device=self.device)
        bad = torch.zeros((1,), dtype=torch.int32, device=self.device)
        nat.check(nat.lib().mi_pack_sparse(d_idx.data_ptr(), d_ptr.data_ptr(), n, m, words.data_ptr(),
                                           bad.data_ptr(), _stream_ptr(self.device)),
                  "mi_pack_sparse")
        if int(bad.item()) != 0:
            raise DomainError(f"row index out of range [0, {n})")
        return words

    def upload(self, words: np.ndarray) -> torch.Tensor:
        """Host words (m, nw) uint64 -> device tensor (int64 storage, same bits)."""
        host = torch.from_numpy(np.ascontiguousarray(words).view(np.int64))
        return host.to(self.device, non_blocking=False)

    def _check_words(self, words_dev: torch.Tensor, n_rows: int, n_cols: int) -> None:
        nw = n_words(n_rows)
        if words_dev.device != self.device or words_dev.dtype not in (torch.int64, torch.uint64):
            raise DimensionError("words must be a 64-bit tensor on the engine's device")
        if tuple(words_dev.shape) != (n_cols, nw) or not words_dev.is_contiguous():
            raise DimensionError(f"words must be contiguous with shape {(n_cols, nw)}")

    def column_order(self, words_dev: torch.Tensor, n_rows: int, n_cols: int,
                     spread: torch.Tensor | None = None) -> tuple[torch.Tensor, torch.Tensor]:
        """(perm, inv): operand slots ordered by column sum (mi_column_order)."""
        self._check_words(words_dev, n_rows, n_cols)
        perm = torch.empty((n_cols,), dtype=torch.int32, device=self.device)
        inv = torch.empty((n_cols,), dtype=torch.int32, device=self.device)
        nat.check(nat.lib().mi_column_order(words_dev.data_ptr(), n_rows, n_cols, perm.data_ptr(), inv.data_ptr(),
                                            spread.data_ptr() if spread is not None else None,
                                            _stream_ptr(self.device)),
                  "mi_column_order")
        return perm, inv

    def choose_order(self, words_dev: torch.Tensor, n_rows: int, n_cols: int, world: int = 1) -> str:
        """The "auto" rule: "colsum" when the column sums are spread wider than
        the table path's per-tile threshold (so natural-order tiles fall back to
        the FP64 epilogue) and m >= AUTO_ORDER_MIN_COLS on one GPU; "natural"
        otherwise.  Below that width the fixed costs (the sort, the m^2
        unpermute pass) outweigh the epilogue saving ("Column
        order").  Reads two integers back (one stream sync)."""
        if world > 1 or n_cols < AUTO_ORDER_MIN_COLS or n_cols <= int(nat.lib().mi_tile_size()):
            return "natural"
        spread = torch.empty((2,), dtype=torch.int32, device=self.device)
        self.column_order(words_dev, n_rows, n_cols, spread)
        lo, hi = (int(x) for x in spread.cpu())
        return "colsum" if hi - lo > nat.get_tuning("table_thr") else "natural"

    @staticmethod
    def words_operand(n_rows: int, n_cols: int) -> bool:
        """The C ABI's rule (mi_words_operand; knobs "xp", "xp_cols"): the
        word-operand GEMM, which expands the packed words in its producer warps
        so that X never reaches HBM, for narrow m (tall-N shapes, where the X
        round trip costs as much as the MMAs)."""
        return bool(nat.lib().mi_words_operand(n_rows, n_cols))

    def _alloc_prepared(self, n_rows: int, n_cols: int, xp: bool = False):
        ld, m_pad = self.layout(n_rows, n_cols)
        x = None if xp else torch.empty((m_pad, ld), dtype=torch.int8, device=self.device)
        colsum = torch.empty((m_pad,), dtype=torch.int32, device=self.device)
        colstat = torch.empty((int(nat.lib().mi_colstat_bytes(n_rows, n_cols)),), dtype=torch.uint8, device=self.device)
        return x, colsum, colstat

    def _rank_mask(self, n_cols: int, rank: int, world: int) -> torch.Tensor | None:
        if world <= 1:
            return None
        key = ("blocks", n_cols, rank, world, nat.get_tuning("cta_group"), nat.get_tuning("band"),
               nat.get_tuning("shard"))
        mask = self._tiles.get(key)
        if mask is None:
            mask = torch.from_numpy(nat.rank_blocks(n_cols, rank, world)).to(self.device)
            self._tiles[key] = mask
        return mask

    def prepare_begin(self, n_rows: int, n_cols: int) -> Prepared:
        """Staged kernel 1, first part (mi_unpack_prep): buffers and the
        per-call prologue; then prepare_range() per column group as its words
        arrive (dispatch's staged broadcast)."""
        xp = self.words_operand(n_rows, n_cols)
        x, colsum, colstat = self._alloc_prepared(n_rows, n_cols, xp)
        ld, m_pad = self.layout(n_rows, n_cols)
        nat.check(nat.lib().mi_unpack_prep(n_rows, n_cols, colstat.data_ptr(), _stream_ptr(self.device)),
                  "mi_unpack_prep")
        return Prepared(n_rows, n_cols, ld, m_pad, x, colsum, colstat)

    def prepare_range(self, prep: Prepared, words_dev: torch.Tensor, c_begin: int, c_end: int,
                      rank: int = 0, world: int = 1) -> None:
        """Expand columns [c_begin, c_end) of X (only rank's blocks when world >
        1) and their statistics (mi_unpack_colsum_range)."""
        self._check_words(words_dev, prep.n_rows, prep.n_cols)
        mask = self._rank_mask(prep.n_cols, rank, world)
        if prep.x is None:  # word-operand path: statistics only, the GEMM reads these words
            prep.words = words_dev
        nat.check(nat.lib().mi_unpack_colsum_range(words_dev.data_ptr(), prep.n_rows, prep.n_cols,
                                                   prep.x.data_ptr() if prep.x is not None else None,
                                                   prep.ld, prep.colstat.data_ptr(), prep.colsum.data_ptr(),
                                                   mask.data_ptr() if mask is not None and prep.x is not None
                                                   else None, c_begin, c_end,
                                                   _stream_ptr(self.device)),
                  "mi_unpack_colsum_range")

    def prepare(self, words_dev: torch.Tensor, n_rows: int, n_cols: int,
                rank: int = 0, world: int = 1, order: str = "natural") -> Prepared:
        """Kernel 1: unpack the packed columns to the K-major operand and
        count ones per column (binmat.column_sums).  With world > 1 only the
        column blocks of rank's tiles are expanded (mi_rank_blocks).
        ``order``: "natural" (slot c = column c), "colsum" (slots ordered by
        column sum, one GPU only; compute() restores column order), or "auto"
        (choose_order)."""
        if order not in ORDERS:
            raise DomainError(f"order must be one of {ORDERS}, got {order!r}")
        self._check_words(words_dev, n_rows, n_cols)
        if order == "auto":
            order = self.choose_order(words_dev, n_rows, n_cols, world)
        if order == "colsum" and world > 1:
            raise DomainError("order='colsum' is single-GPU only (each rank would unpermute the whole matrix)")
        ld, m_pad = self.layout(n_rows, n_cols)
        if order == "natural" and self.words_operand(n_rows, n_cols):
            # word-operand path: nothing to expand; the first compute() also
            # computes the column statistics (mi_gram_mi_words_stats: inside the
            # fused launch for the full tile list of a narrow matrix)
            x, colsum, colstat = self._alloc_prepared(n_rows, n_cols, True)
            return Prepared(n_rows, n_cols, ld, m_pad, None, colsum, colstat, words=words_dev, stats_ready=False)
        x, colsum, colstat = self._alloc_prepared(n_rows, n_cols)
        mask = self._rank_mask(n_cols, rank, world)
        if order == "colsum":
            perm, inv = self.column_order(words_dev, n_rows, n_cols)
            nat.check(nat.lib().mi_unpack_colsum_ordered(words_dev.data_ptr(), n_rows, n_cols, perm.data_ptr(),
                                                         x.data_ptr(), ld, colstat.data_ptr(), colsum.data_ptr(),
                                                         _stream_ptr(self.device)),
                      "mi_unpack_colsum_ordered")
            return Prepared(n_rows, n_cols, ld, m_pad, x, colsum, colstat, perm, inv)
        nat.check(nat.lib().mi_unpack_colsum_blocks(words_dev.data_ptr(), n_rows, n_cols, x.data_ptr(), ld,
                                                    colstat.data_ptr(), colsum.data_ptr(),
                                                    mask.data_ptr() if mask is not None else None,
                                                    _stream_ptr(self.device)),
                  "mi_unpack_colsum_blocks")
        return Prepared(n_rows, n_cols, ld, m_pad, x, colsum, colstat)

    def compute(self, prep: Prepared, cfg=None, out_dtype: torch.dtype = torch.float64,
                tiles: torch.Tensor | None = None, out: torch.Tensor | None = None,
                packed: bool = False, tile_major: bool = False) -> torch.Tensor:
        """Kernels 2+3: fused Gram + MI over `tiles` (all upper-triangle tiles by
        default), each written with its mirror into `out` (m x m) -- or, with
        ``packed``, only j >= i into a flat m(m+1)/2 tensor (row-major upper
        triangle; ``unpack_upper`` restores the square) -- or, with
        ``tile_major``, tile k alone into out[k] (k x TS x TS; the sharded form
        of dispatch.Shard)."""
        if out_dtype not in _OUT_KIND:
            raise DomainError(f"out_dtype must be float64, float32 or int32, got {out_dtype}")
        mode, eps, diag = _config_fields(cfg)
        kind = _OUT_KIND[out_dtype]
        if kind == nat.MI_OUT_COUNTS:
            mode = nat.MI_MODE_EXACT
        m = prep.n_cols
        if prep.layout_knobs != _layout_knobs():
            raise DomainError("the fp4 / cta_group knobs changed between prepare() and compute(): "
                              f"X was laid out for {prep.layout_knobs}, the kernel would read {_layout_knobs()}")
        if prep.perm is not None:
            if tile_major:
                raise DomainError("order='colsum' computes the full matrix: no tile-major output")
            return self._compute_ordered(prep, mode, eps, diag, kind, out_dtype, tiles, out, packed)
        if tile_major:
            if tiles is None:
                tiles = self.tiles(m)
            ts = int(nat.lib().mi_tile_size())
            k = int(tiles.shape[0])
            if out is None:
                out = torch.empty((max(k, 1), ts, ts), dtype=out_dtype, device=self.device)
            if out.dtype != out_dtype or out.dim() != 3 or out.shape[0] < k or tuple(out.shape[1:]) != (ts, ts) \
                    or not out.is_contiguous() or out.device != self.device:
                raise DimensionError("tile-major out must be a contiguous (>= k, TS, TS) tensor of out_dtype")
            ld_out = nat.MI_TILE_MAJOR
        elif packed:
            if out is None:
                out = torch.empty((m * (m + 1) // 2,), dtype=out_dtype, device=self.device)
            if out.dtype != out_dtype or out.dim() != 1 or out.numel() < m * (m + 1) // 2 or out.stride(0) != 1 \
                    or out.device != self.device:
                raise DimensionError("packed out must be a flat m(m+1)/2 tensor of out_dtype on the device")
            ld_out = nat.MI_PACKED_UPPER
        else:
            if out is None:
                out = torch.empty((m, m), dtype=out_dtype, device=self.device)
            if out.dtype != out_dtype or out.dim() != 2 or out.shape[0] < m or out.shape[1] < m \
                    or out.stride(1) != 1 or out.device != self.device:
                raise DimensionError("out must be a row-major (>= m, >= m) tensor of out_dtype on the device")
            ld_out = out.stride(0)
        if tiles is None:
            tiles = self.tiles(m)
        if prep.x is None:
            if prep.words is None:
                raise DomainError("word-operand prepare without words (prepare_range was not called)")
            if prep.stats_ready:
                nat.check(nat.lib().mi_gram_mi_words(prep.words.data_ptr(), prep.colstat.data_ptr(), prep.n_rows, m,
                                                     mode, eps, diag, kind, out.data_ptr(), ld_out,
                                                     tiles.data_ptr(), tiles.shape[0], _stream_ptr(self.device)),
                          "mi_gram_mi_words")
            else:
                nat.check(nat.lib().mi_gram_mi_words_stats(prep.words.data_ptr(), prep.colstat.data_ptr(),
                                                           prep.colsum.data_ptr(), prep.n_rows, m, mode, eps, diag,
                                                           kind, out.data_ptr(), ld_out, tiles.data_ptr(),
                                                           tiles.shape[0], _stream_ptr(self.device)),
                          "mi_gram_mi_words_stats")
                prep.stats_ready = True
            return out
        nat.check(nat.lib().mi_gram_mi(prep.x.data_ptr(), prep.colstat.data_ptr(), prep.n_rows, m, prep.ld,
                                       mode, eps, diag, kind, out.data_ptr(), ld_out,
                                       tiles.data_ptr(), tiles.shape[0], _stream_ptr(self.device)),
                  "mi_gram_mi")
        return out

    def _compute_ordered(self, prep: Prepared, mode: int, eps: float, diag: int, kind: int,
                         out_dtype: torch.dtype, tiles, out, packed: bool) -> torch.Tensor:
        """Column-sum order: the fused kernel writes the full matrix in slot
        order into a scratch matrix, mi_unpermute puts it back in column order."""
        if packed or tiles is not None:
            raise DomainError("order='colsum' computes the full matrix: no packed output or tile subsets")
        m = prep.n_cols
        if out is None:
            out = torch.empty((m, m), dtype=out_dtype, device=self.device)
        if out.dtype != out_dtype or out.dim() != 2 or out.shape[0] < m or out.shape[1] < m \
                or out.stride(1) != 1 or out.device != self.device:
            raise DimensionError("out must be a row-major (>= m, >= m) tensor of out_dtype on the device")
        slot = torch.empty((m, m), dtype=out_dtype, device=self.device)
        stream = _stream_ptr(self.device)
        tl = self.tiles(m)
        nat.check(nat.lib().mi_gram_mi(prep.x.data_ptr(), prep.colstat.data_ptr(), prep.n_rows, m, prep.ld,
                                       mode, eps, diag, kind, slot.data_ptr(), m, tl.data_ptr(), tl.shape[0],
                                       stream),
                  "mi_gram_mi")
        nat.check(nat.lib().mi_unpermute(slot.data_ptr(), m, out.data_ptr(), out.stride(0), m, slot.element_size(),
                                         prep.inv.data_ptr(), stream),
                  "mi_unpermute")
        return out

    def compute_slot_order(self, prep: Prepared, cfg=None, out_dtype: torch.dtype = torch.float64,
                           out: torch.Tensor | None = None) -> tuple[torch.Tensor, torch.Tensor]:
        """The column-sum-ordered result without the unpermute pass: (S, perm)
        with S[a, b] = MI(perm[a], perm[b]).  For consumers that only need
        pairs and their values (thresholds, top-k), this skips the m^2 pass
        (config 4: 19.5 ms of fused kernel instead of 19.5 + 4.6)."""
        if prep.perm is None:
            raise DomainError("compute_slot_order needs a prepare(order='colsum') operand")
        if out_dtype not in _OUT_KIND:
            raise DomainError(f"out_dtype must be float64, float32 or int32, got {out_dtype}")
        mode, eps, diag = _config_fields(cfg)
        kind = _OUT_KIND[out_dtype]
        if kind == nat.MI_OUT_COUNTS:
            mode = nat.MI_MODE_EXACT
        m = prep.n_cols
        if out is None:
            out = torch.empty((m, m), dtype=out_dtype, device=self.device)
        if out.dtype != out_dtype or out.dim() != 2 or out.shape[0] < m or out.shape[1] < m \
                or out.stride(1) != 1 or out.device != self.device:
            raise DimensionError("out must be a row-major (>= m, >= m) tensor of out_dtype on the device")
        tl = self.tiles(m)
        nat.check(nat.lib().mi_gram_mi(prep.x.data_ptr(), prep.colstat.data_ptr(), prep.n_rows, m, prep.ld,
                                       mode, eps, diag, kind, out.data_ptr(), out.stride(0), tl.data_ptr(),
                                       tl.shape[0], _stream_ptr(self.device)),
                  "mi_gram_mi")
        return out, prep.perm

    # ------------------------------------------------------------------ composites
    def all_pairs_device(self, words_dev: torch.Tensor, n_rows: int, n_cols: int, cfg=None,
                         out_dtype: torch.dtype = torch.float64, out: torch.Tensor | None = None,
                         order: str = "natural") -> torch.Tensor:
        """Device words in, device MI (m x m, column order) out.  ``order``:
        see prepare() ("natural" keeps results bit-identical to the
        multi-GPU path's)."""
        return self.compute(self.prepare(words_dev, n_rows, n_cols, order=order), cfg, out_dtype, out=out)

    def all_pairs_bmi(self, path, cfg=None, out_dtype: torch.dtype = torch.float64) -> torch.Tensor:
        """MI straight from a BMI1 file (the reference's packed container,
        io.py:1-16): payload streamed to the device, then kernels 1-3."""
        from .io import read_bmi_device

        words, n_rows, n_cols = read_bmi_device(path, self.device)
        return self.all_pairs_device(words, n_rows, n_cols, cfg, out_dtype)

    def gram_counts(self, words_dev: torch.Tensor, n_rows: int, n_cols: int) -> tuple[torch.Tensor, torch.Tensor]:
        """Debug export for parity: (G11 int32 m x m, column sums int32 m)."""
        prep = self.prepare(words_dev, n_rows, n_cols)
        g = self.compute(prep, None, torch.int32)
        return g, prep.colsum[:n_cols]

    def all_pairs_host(self, words: np.ndarray | torch.Tensor, n_rows: int, n_cols: int, cfg=None,
                       out_dtype: torch.dtype = torch.float64, host_out: torch.Tensor | None = None,
                       packed: bool = False) -> torch.Tensor:
        """Host words in, host MI out, through the C ABI's mi_all_pairs_host:
        H2D, kernel 1, the fused kernel, and a D2H of finished row bands that
        overlaps the GEMM.  ``host_out``: a pinned CPU tensor / registered
        array (D2H straight into it), or pageable memory (numpy: filled
        through the library's pinned egress buffer by host copy threads); by
        default a fresh numpy array.
        ``packed``: the upper triangle only (mi_all_pairs_host_packed), a flat
        m(m+1)/2 tensor -- half the device-to-host bytes."""
        mode, eps, diag = _config_fields(cfg)
        if out_dtype not in (torch.float64, torch.float32):
            raise DomainError(f"out_dtype must be float64 or float32, got {out_dtype}")
        if isinstance(words, torch.Tensor):
            if words.device.type != "cpu" or not words.is_contiguous() or words.element_size() != 8:
                raise DimensionError("host words must be a contiguous 64-bit CPU tensor")
            if tuple(words.shape) != (n_cols, n_words(n_rows)):
                raise DimensionError(f"words must have shape {(n_cols, n_words(n_rows))}")
            wptr, keep = words.data_ptr(), words
        else:
            keep = np.ascontiguousarray(words)
            if keep.dtype != np.uint64 or keep.shape != (n_cols, n_words(n_rows)):
                raise DimensionError(f"words must be uint64 with shape {(n_cols, n_words(n_rows))}")
            wptr = keep.ctypes.data
        shape = (n_cols * (n_cols + 1) // 2,) if packed else (n_cols, n_cols)
        np_dt = np.float64 if out_dtype == torch.float64 else np.float32
        if host_out is None:
            # ordinary (pageable) memory owned by the caller: the C ABI fills it
            # through its cached pinned egress buffer, piece by piece
            host_out = np.empty(shape, dtype=np_dt)
        if isinstance(host_out, np.ndarray):
            if host_out.dtype != np_dt or tuple(host_out.shape) != shape or not host_out.flags.c_contiguous:
                raise DimensionError(f"host_out must be a C-contiguous {shape} {np.dtype(np_dt).name} array")
            out_ptr = host_out.ctypes.data
        else:
            if host_out.dtype != out_dtype or tuple(host_out.shape) != shape or not host_out.is_contiguous() \
                    or host_out.device.type != "cpu":
                raise DimensionError(f"host_out must be a contiguous {shape} CPU tensor of out_dtype")
            out_ptr = host_out.data_ptr()
        kind = nat.MI_OUT_F64 if out_dtype == torch.float64 else nat.MI_OUT_F32
        fn = nat.lib().mi_all_pairs_host_packed if packed else nat.lib().mi_all_pairs_host
        nat.check(fn(wptr, n_rows, n_cols, mode, eps, diag, kind, out_ptr, self.device.index), "mi_all_pairs_host")
        del keep
        return host_out


def _host_words(data, device: int | None = None) -> tuple[int, int, np.ndarray]:
    """(n_rows, n_cols, words) of any input: dense words as they are; the
    sparse backend's index lists packed on the GPU (MIEngine.from_sparse)."""
    if not hasattr(data, "words") and hasattr(data, "col_indices"):
        w = MIEngine.get(device).from_sparse(data)
        return int(data.n_rows), int(data.n_cols), w.cpu().numpy().view(np.uint64)
    return as_dense_words(data)


def mi_all_pairs(data, cfg: EngineConfig | None = None, backend: str = "dense", threads: int = 0,
                 device: int | None = None, devices=None) -> MIMatrix:
    """Full pairwise MI matrix (drop-in for engine.mi_all_pairs, engine.py:144-168).

    ``backend`` must be one of the reference's names ("dense", "sparse",
    "direct"); all run the same GPU path.  ``threads`` is accepted and ignored:
    results are bit-identical regardless of parallelism.  ``devices``: a list
    of GPU indices to share the work in this process (mi_all_pairs_devices).
    """
    if backend not in BACKENDS:
        raise DomainError(f"backend must be one of {BACKENDS}, got {backend!r}")
    _config_fields(cfg)
    if devices is not None and len(devices) > 1:
        return MIMatrix(values=mi_all_pairs_devices(data, devices, cfg))
    n, m, words = _host_words(data, device if devices is None else devices[0])
    eng = MIEngine.get(device if devices is None else devices[0])
    values = np.empty((m, m), dtype=np.float64)  # fresh, caller-owned, like the reference's
    eng.all_pairs_host(words, n, m, cfg, torch.float64, host_out=values)
    return MIMatrix(values=values)


def mi_all_pairs_devices(data, devices, cfg: EngineConfig | None = None, out_dtype=np.float64,
                         out: np.ndarray | None = None) -> np.ndarray:
    """The full matrix from several GPUs of this process (C ABI
    mi_all_pairs_host_devices): the triangle's tiles are dealt as over the
    ranks of the multi-GPU path, each device uploads the words and writes its
    tiles and mirrors into the host matrix over its own link (zero copy when
    ``out`` is pinned and mapped, e.g. registered with mi_host_register).  A
    device may be listed more than once (it then runs several shares)."""
    mode, eps, diag = _config_fields(cfg)
    n, m, words = _host_words(data, int(list(devices)[0]) if len(list(devices)) else None)
    devs = np.ascontiguousarray(np.asarray(list(devices), dtype=np.int32))
    if devs.ndim != 1 or devs.size < 1:
        raise DomainError("devices must be a non-empty list of GPU indices")
    if out is None:
        out = np.empty((m, m), dtype=out_dtype)
    if out.dtype not in (np.float64, np.float32) or out.shape != (m, m) or not out.flags.c_contiguous:
        raise DimensionError(f"out must be a C-contiguous ({m}, {m}) float64 or float32 array")
    kind = nat.MI_OUT_F64 if out.dtype == np.float64 else nat.MI_OUT_F32
    w = np.ascontiguousarray(words)
    nat.check(nat.lib().mi_all_pairs_host_devices(w.ctypes.data, n, m, mode, eps, diag, kind, out.ctypes.data,
                                                  devs.ctypes.data, int(devs.size)),
              "mi_all_pairs_host_devices")
    return out


def unpack_upper(packed, m: int):
    """Square symmetric (m, m) matrix from the packed upper triangle
    (MI_PACKED_UPPER layout: row i holds columns i..m-1).  numpy or torch."""
    iu = np.triu_indices(m)
    if isinstance(packed, torch.Tensor):
        out = torch.empty((m, m), dtype=packed.dtype, device=packed.device)
        r = torch.from_numpy(iu[0]).to(packed.device)
        c = torch.from_numpy(iu[1]).to(packed.device)
        out[r, c] = packed
        out[c, r] = packed
        return out
    out = np.empty((m, m), dtype=packed.dtype)
    out[iu] = packed
    out.T[iu] = packed
    return out


def gram_ones(data, device: int | None = None) -> np.ndarray:
    """Drop-in for gram.gram_ones (gram.py:56-65): int64 m x m co-occurring ones."""
    n, m, words = _host_words(data, device)
    out = np.empty((m, m), dtype=np.int64)
    w = np.ascontiguousarray(words)
    dev = MIEngine.get(device).device.index
    nat.check(nat.lib().mi_gram_ones_host(w.ctypes.data, m, w.shape[1], out.ctypes.data, dev), "mi_gram_ones_host")
    return out


def column_sums(data, device: int | None = None) -> np.ndarray:
    """Drop-in for binmat.column_sums (binmat.py:175-177), computed by kernel 1."""
    n, m, words = _host_words(data, device)
    out = np.empty((m,), dtype=np.uint64)
    w = np.ascontiguousarray(words)
    dev = MIEngine.get(device).device.index
    nat.check(nat.lib().mi_column_sums_host(w.ctypes.data, m, w.shape[1], out.ctypes.data, dev),
              "mi_column_sums_host")
    return out


def mi_all_pairs_c_abi(data, cfg: EngineConfig | None = None, device: int = 0,
                       out_dtype=np.float64) -> np.ndarray:
    """Same computation through the pure C entry point mi_all_pairs_host (what a
    non-Python binding would call); used by tests and the e2e cross-check."""
    mode, eps, diag = _config_fields(cfg)
    n, m, words = _host_words(data, device)
    out = np.empty((m, m), dtype=out_dtype)
    kind = nat.MI_OUT_F64 if out_dtype == np.float64 else nat.MI_OUT_F32
    w = np.ascontiguousarray(words)
    nat.check(nat.lib().mi_all_pairs_host(w.ctypes.data, n, m, mode, eps, diag, kind, out.ctypes.data, device),
              "mi_all_pairs_host")
    return out

