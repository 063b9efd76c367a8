/*
 * mimatrix_b200.h -- C ABI of the B200-native all-pairs binary mutual
 * information engine (libmimatrix_b200.so).
 *
 * Plain pointers and sizes only; no torch or CUDA C++ types in the
 * signatures (`stream` is a cudaStream_t passed as void*, NULL = default).
 * Every function returns MI_OK (0) or an MI_ERR_* code; the message for the
 * last failure on the calling thread is available from mi_last_error().
 *
 * Reference interfaces replaced (paths relative to
 * /root/reference/pkg/src/mimatrix/):
 *   mi_all_pairs_host   engine.py:144-168   mi_all_pairs(data, cfg, backend, threads)
 *                                           (dense path; float64 m x m result)
 *   mi_gram_ones_host   _kernels.py:48-61   gram_ones_kernel(words, out) / gram.py:56-65
 *   mi_column_sums_host binmat.py:175-177   column_sums(matrix)
 *   mi_unpack_colsum    binmat.py:175-177 + the per-column word streams that
 *                                           _kernels.py:36-45 reads
 *   mi_gram_mi          _kernels.py:48-61 + gram.py:88-111 + engine.py:93-141
 *                                           (G11, closed-form counts, MI; fused)
 *   mi_generate_words   datagen.py:44-73    generate(GenSpec) stream, packed
 *   mi_pack_bits        binmat.py:34-46,136-172  from_bits / from_rows (pack_bits), on the device
 *   mi_bmi_header,      io.py:92-116        read_bmi(path) (BMI1 container, io.py:1-16),
 *   mi_bmi_load                             payload streamed straight to the device
 * Extensions with no reference counterpart: mi_all_pairs_host_packed and
 * ld_out = MI_PACKED_UPPER (upper-triangle egress), mi_tile_list /
 * mi_rank_blocks / mi_unpack_colsum_blocks (multi-GPU shares),
 * mi_column_order / mi_unpack_colsum_ordered / mi_unpermute (column-sum order),
 * mi_host_register / mi_copy_tiles_to_host / mi_scatter_tiles and
 * ld_out = MI_TILE_MAJOR (sharded output and its gather), the
 * layout queries and the tuning knobs.
 * Error codes mirror the reference's exception classes (errors.py:8-25).
 */
#ifndef MIMATRIX_B200_H
#define MIMATRIX_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MI_B200_ABI_VERSION 1

/* return codes (errors.py:8-25) */
#define MI_OK 0
#define MI_ERR_DIMENSION 1   /* DimensionError   */
#define MI_ERR_DOMAIN 2      /* DomainError      */
#define MI_ERR_CONSISTENCY 3 /* ConsistencyError */
#define MI_ERR_CUDA 4        /* device / driver failure (MiMatrixError) */
#define MI_ERR_UNSUPPORTED 5 /* not an sm_100 device, or no device   */
#define MI_ERR_FORMAT 6      /* FormatError (a malformed BMI1 file)  */

/* ld_out value selecting the packed upper-triangle output: element (i, j >= i)
 * at i*m - i*(i-1)/2 + (j - i), m(m+1)/2 elements, nothing mirrored. */
#define MI_PACKED_UPPER 0
/* ld_out value selecting the tile-major (sharded) output of mi_gram_mi: tile k
 * of the launch's list is stored at d_out + k * T * T elements (T =
 * mi_tile_size(), row pitch T, element (i, j) of tile (I, J) at row i - I*T,
 * column j - J*T), without its mirror.  mi_scatter_tiles places such shards
 * (tiles and mirrors) into a full matrix on a device or in pinned host memory. */
#define MI_TILE_MAJOR (-1)

/* engine modes (engine.py:28, EngineConfig.mode) */
#define MI_MODE_EXACT 0
#define MI_MODE_EPSILON 1

/* output kinds for mi_gram_mi / mi_all_pairs_host */
#define MI_OUT_COUNTS 0 /* int32 G11 (debug export, bit-exact parity)  */
#define MI_OUT_F64 1    /* float64 MI (the reference's MIMatrix.values) */
#define MI_OUT_F32 2    /* float32 MI (device API, 1e-6 contract)       */

int mi_b200_abi_version(void);
const char* mi_last_error(void);
/* number of SMs and compute capability of `device`; MI_ERR_UNSUPPORTED if absent */
int mi_device_info(int device, int* num_sms, int* cc_major, int* cc_minor);

/* ---- layout helpers (host only, no device needed) ---- */
/* bytes per operand row ("ld") of the K-major operand written by
 * mi_unpack_colsum and read by mi_gram_mi.  The operand is stored k-blocked,
 * [ld/128][m_pad][128 bytes].  Format (fixed by n_rows and the "fp4" /
 * "cta_group" knobs, which must not change between the two calls):
 *   e2m1 (default: n_rows < 2^24, SM-pair tiles): row r of column c is the
 *     nibble (r % 2) of byte ((r/256) * m_pad + c) * 128 + (r % 256) / 2,
 *     0 or 1.0 (0b0010); ld = roundup(n_rows, 256) / 2;
 *   int8 (otherwise): byte ((r/128) * m_pad + c) * 128 + r % 128 is 0 or 1;
 *     ld = roundup(n_rows, 128). */
int64_t mi_kmajor_ld(int64_t n_rows);
/* padded column count m_pad (operand rows, multiple of the tile size) */
int64_t mi_kmajor_rows(int64_t n_cols);
/* bytes of the per-column statistics workspace that kernel 1 writes and the
 * fused kernel reads: marginal counts, their log2 splits and fixed-point
 * c*log2(c) marginal terms */
int64_t mi_colstat_bytes(int64_t n_rows, int64_t n_cols);
/* output tile edge (256: a 2-SM tcgen05 tile) */
int mi_tile_size(void);
/* number of upper-triangle tiles (I <= J) for m columns */
int64_t mi_num_tiles(int64_t n_cols);
/* Fill `tiles_out` with the (I, J) pairs (int32 x 2 each) that rank `rank` of
 * `world` computes, in L2-friendly banded order (`band` tile rows per band,
 * <= 0 for the default).  Returns the count (or -MI_ERR_* on error); pass
 * tiles_out = NULL to query the count. */
int64_t mi_tile_list(int64_t n_cols, int rank, int world, int band, int32_t* tiles_out,
                     int64_t capacity);
/* the column blocks (of mi_tile_size() columns) rank's tiles touch: mask_out[b]
 * = 1/0 for b < ceil(n_cols / tile); returns the number of marked blocks, or
 * the block count when mask_out = NULL (8 ranks: half of them, see the
 * "shard" knob; other world sizes: nearly all). */
int64_t mi_rank_blocks(int64_t n_cols, int rank, int world, uint8_t* mask_out, int64_t capacity);

/* ---- device-pointer entry points, enqueued on `stream` ---- */
/* words (m x nw uint64, nw = ceil(n_rows/64)) -> kmajor (k-blocked, m_pad * ld int8),
 * d_colstat (mi_colstat_bytes) and, if d_colsum != NULL, the column sums
 * (m_pad int32; padding columns get 0). */
int mi_unpack_colsum(const uint64_t* d_words, int64_t n_rows, int64_t n_cols, int8_t* d_kmajor,
                     int64_t ld, void* d_colstat, int32_t* d_colsum, void* stream);
/* the same, expanding only the column blocks marked in d_block_mask (device,
 * one byte per block as from mi_rank_blocks; NULL = all): a rank's share of X.
 * Statistics of unmarked columns are not meaningful. */
int mi_unpack_colsum_blocks(const uint64_t* d_words, int64_t n_rows, int64_t n_cols, int8_t* d_kmajor,
                            int64_t ld, void* d_colstat, int32_t* d_colsum, const uint8_t* d_block_mask,
                            void* stream);
/* mi_unpack_colsum_blocks in pieces, for staged ingest (words arriving by
 * column groups): mi_unpack_prep once (per-column counters, block ranges, the
 * fixed-point table), then mi_unpack_colsum_range for columns [c_begin, c_end)
 * (c_begin and c_end multiples of 32, c_end <= mi_kmajor_rows(n_cols)) once their
 * words are on the device; the ranges must cover every column before the
 * tiles that need them run. */
int mi_unpack_prep(int64_t n_rows, int64_t n_cols, void* d_colstat, void* stream);
int mi_unpack_colsum_range(const uint64_t* d_words, int64_t n_rows, int64_t n_cols, int8_t* d_kmajor,
                           int64_t ld, void* d_colstat, int32_t* d_colsum, const uint8_t* d_block_mask,
                           int64_t c_begin, int64_t c_end, void* stream);
/* Fused G11 + MI over the listed upper-triangle tiles; writes each tile and
 * its mirror into d_out (row-major, pitch ld_out elements), or with ld_out =
 * MI_PACKED_UPPER only the elements j >= i, packed, or with ld_out =
 * MI_TILE_MAJOR each tile alone into its slot (see above). */
int mi_gram_mi(const int8_t* d_kmajor, const void* d_colstat, int64_t n_rows, int64_t n_cols,
               int64_t ld, int mode, double epsilon, int include_diagonal, int out_kind, void* d_out,
               int64_t ld_out, const int32_t* d_tiles, int64_t n_tiles, void* stream);
/* ---- word-operand path (tall-N / narrow-m) ----
 * The same fused Gram + MI, reading the packed words themselves (the
 * reference's gram_ones_kernel reads them too, _kernels.py:36-45): producer
 * warps expand each k-block of 256 rows into the swizzled shared-memory
 * stages, so the e2m1 operand X never exists in HBM (for narrow m its write
 * and read-back cost more than the MMAs).  d_colstat comes from
 * mi_colstat_words (column sums and statistics only: one read of the words,
 * no expansion).  Needs e2m1 operands (n_rows < 2^24, SM-pair tiles).
 * Same outputs, tile lists and ld_out forms as mi_gram_mi; bit-identical. */
/* 1 when the engine's rule ("xp" / "xp_cols" knobs) picks the word-operand
 * path for this shape, else 0 (the unpack + TMA path). */
int mi_words_operand(int64_t n_rows, int64_t n_cols);
int mi_colstat_words(const uint64_t* d_words, int64_t n_rows, int64_t n_cols, void* d_colstat, int32_t* d_colsum,
                     void* stream);
int mi_gram_mi_words(const uint64_t* d_words, const void* d_colstat, int64_t n_rows, int64_t n_cols, int mode,
                     double epsilon, int include_diagonal, int out_kind, void* d_out, int64_t ld_out,
                     const int32_t* d_tiles, int64_t n_tiles, void* stream);
/* mi_gram_mi_words that also computes the column statistics into d_colstat
 * (and the column sums into d_colsum, if not NULL): no mi_colstat_words
 * first.  With the full tile list of a narrow matrix (every tile a K-range
 * tail unit: the default schedule when the tiles are fewer than the SM pairs)
 * it is ONE fused launch that reads the words once -- the expander warps count
 * the ones of each column on the diagonal tiles' units and the epilogue warps
 * build the statistics while the units run ("xp_stats" knob, default 1);
 * otherwise kernel 1's counting pass runs first. */
int mi_gram_mi_words_stats(const uint64_t* d_words, void* d_colstat, int32_t* d_colsum, int64_t n_rows,
                           int64_t n_cols, int mode, double epsilon, int include_diagonal, int out_kind, void* d_out,
                           int64_t ld_out, const int32_t* d_tiles, int64_t n_tiles, void* stream);
/* binmat.from_bits / from_rows (binmat.py:34-46,136-172) on the device: a
 * row-major uint8 0/1 matrix (n_rows x n_cols, row pitch ld_bits bytes) ->
 * the words layout (n_cols x ceil(n_rows/64) uint64, padding bits zero).
 * *d_bad (device int32, zeroed by the caller) gets bit 0 set if any byte is
 * neither 0 nor 1 (from_rows's DomainError); the words are then not valid. */
int mi_pack_bits(const uint8_t* d_bits, int64_t n_rows, int64_t n_cols, int64_t ld_bits, uint64_t* d_words,
                 int32_t* d_bad, void* stream);
/* binmat.to_dense (binmat.py:187-194) on the device, for the sparse backend's
 * SparseBinaryMatrix (per-column row-index lists, binmat.py:100-133): CSC
 * arrays d_indptr[n_cols + 1] (int64 offsets into d_indices) and d_indices
 * (int64 row indices) -> the words layout (zeroed, then the bits set; cost ~
 * nnz).  *d_bad (device int32, zeroed by the caller) gets bit 0 set for an
 * index outside [0, n_rows) (the words are then not valid). */
int mi_pack_sparse(const int64_t* d_indices, const int64_t* d_indptr, int64_t n_rows, int64_t n_cols,
                   uint64_t* d_words, int32_t* d_bad, void* stream);
/* ---- column order by column sum (configs with spread densities) ----
 * The fused epilogue's FP64-free table path needs each tile's column sums to
 * be clustered; computing in slots ordered by column sum makes that true for
 * spread densities, and mi_unpermute restores column order afterwards.
 * mi_column_order: d_perm[s] = the column placed in operand slot s (ascending
 * column sum, ties by column index: deterministic), d_inv[c] = slot of column
 * c (n_cols int32 each); d_spread (2 int32, or NULL) = (min, max) column sum. */
int mi_column_order(const uint64_t* d_words, int64_t n_rows, int64_t n_cols, int32_t* d_perm,
                    int32_t* d_inv, int32_t* d_spread, void* stream);
/* mi_unpack_colsum with operand slot s holding column d_perm[s] (NULL =
 * identity); d_colstat / d_colsum are then in slot order. */
int mi_unpack_colsum_ordered(const uint64_t* d_words, int64_t n_rows, int64_t n_cols, const int32_t* d_perm,
                             int8_t* d_kmajor, int64_t ld, void* d_colstat, int32_t* d_colsum, void* stream);
/* d_out[r][c] = d_in[d_inv[r]][d_inv[c]] for r, c < n_cols (pitches in
 * elements of esz = 4 or 8 bytes; d_in and d_out must not overlap): a result
 * computed in slot order (full square, as mi_gram_mi writes it) back in
 * column order.  HBM-bound, one read and one write of the matrix. */
int mi_unpermute(const void* d_in, int64_t ld_in, void* d_out, int64_t ld_out, int64_t n_cols, int esz,
                 const int32_t* d_inv, void* stream);
/* Packed words of a synthetic dataset.  col_kind[c]: 0 Bernoulli(col_threshold[c]),
 * 1 all zero, 2 all one, 3 col_src[c] XOR Bernoulli(flip_threshold) drawn
 * with flip_seed.  Thresholds are ceil(p * 2^64) (datagen.py:53-55). */
int mi_generate_words(uint64_t* d_words, int64_t n_rows, int64_t n_cols, uint64_t seed,
                      const uint64_t* d_col_threshold, const uint8_t* d_col_kind,
                      const int32_t* d_col_src, uint64_t flip_threshold, uint64_t flip_seed,
                      void* stream);

/* ---- host-buffer entry points (H2D, compute, D2H inside; blocking) ---- */
/* engine.mi_all_pairs(dense): h_out is n_cols x n_cols, float64 (MI_OUT_F64)
 * or float32 (MI_OUT_F32). */
int mi_all_pairs_host(const uint64_t* h_words, int64_t n_rows, int64_t n_cols, int mode,
                      double epsilon, int include_diagonal, int out_kind, void* h_out, int device);
/* mi_all_pairs_host on several GPUs of this process (devices[0..n_devices)):
 * the tiles are dealt as over the ranks of the multi-GPU path, every device
 * uploads the words over its own link, computes its share and writes its tiles
 * and mirrors straight into the host matrix over its own link (zero copy into
 * h_out when it is pinned and mapped -- mi_host_register -- else into a cached
 * pinned matrix copied out at the end).  Bit-identical to one device. */
int mi_all_pairs_host_devices(const uint64_t* h_words, int64_t n_rows, int64_t n_cols, int mode, double epsilon,
                              int include_diagonal, int out_kind, void* h_out, const int* devices, int n_devices);
/* the same result as the packed upper triangle (MI_PACKED_UPPER layout,
 * n_cols (n_cols+1)/2 elements in h_out): half the device-to-host bytes */
int mi_all_pairs_host_packed(const uint64_t* h_words, int64_t n_rows, int64_t n_cols, int mode,
                             double epsilon, int include_diagonal, int out_kind, void* h_out, int device);
/* _kernels.gram_ones_kernel(words, out): words is n_cols x n_words; out is
 * n_cols x n_cols int64 (both triangles, diagonal = column sums). */
int mi_gram_ones_host(const uint64_t* h_words, int64_t n_cols, int64_t n_words, int64_t* h_out,
                      int device);
/* binmat.column_sums(matrix) */
int mi_column_sums_host(const uint64_t* h_words, int64_t n_cols, int64_t n_words, uint64_t* h_out,
                        int device);
/* ---- egress of a sharded result into one host matrix ----
 * Pin host memory allocated elsewhere (e.g. a POSIX shared-memory segment
 * that every rank on the node maps) for asynchronous copies and for device
 * kernels writing it directly (mapped, portable). */
int mi_host_register(void* h_ptr, int64_t bytes);
int mi_host_unregister(void* h_ptr);
/* Copy the listed tiles (h_tiles: host (I, J) pairs as from mi_tile_list) and
 * their mirrors from d_out (pitch ld_out elements of esz = 4 or 8 bytes) into
 * h_dst (pitch ld_dst), clipped to n_cols, as merged 2-D copies on `stream`
 * (asynchronous): every rank writes its share of the full matrix over its own
 * PCIe link. */
int mi_copy_tiles_to_host(const void* d_out, int64_t ld_out, int64_t n_cols, int esz, const int32_t* h_tiles,
                          int64_t n_tiles, void* h_dst, int64_t ld_dst, void* stream);
/* Tile-major shards (mi_gram_mi with MI_TILE_MAJOR) -> a full row-major matrix:
 * tile k of d_tiles (device (I, J) pairs) from d_src + k*T*T into rows I*T..,
 * columns J*T.. of d_dst (pitch ld_dst elements, esz 4 or 8 bytes), and with
 * `mirror` its transpose at (J, I) as well (off-diagonal tiles).  d_dst may be
 * device memory or pinned / mi_host_register'ed host memory (written over
 * PCIe by the kernel, zero-copy).  The multi-GPU gather: each rank places its
 * own shard. */
int mi_scatter_tiles(const void* d_src, const int32_t* d_tiles, int64_t n_tiles, int64_t n_cols, int esz, void* d_dst,
                     int64_t ld_dst, int mirror, void* stream);

/* ---- ingest: the BMI1 packed container (io.py:1-16, read_bmi io.py:92-116) ----
 * "BMI1", n_rows (u64 LE), n_cols (u64 LE), then n_cols columns of
 * ceil(n_rows/64) little-endian words -- byte for byte the words layout, so
 * the payload goes to the device as is.
 * mi_bmi_header validates the header and the payload length (MI_ERR_FORMAT,
 * with read_bmi's messages) and returns the shape. */
int mi_bmi_header(const char* path, int64_t* n_rows, int64_t* n_cols);
/* Stream the payload into d_words (n_cols x ceil(n_rows/64) uint64 on the
 * current device) through pinned double-buffered staging, file reads
 * overlapping the H2D copies on `stream`; nonzero padding bits past row
 * n_rows - 1 are rejected (MI_ERR_FORMAT) like read_bmi.  Returns after the
 * last copy completed. */
int mi_bmi_load(const char* path, uint64_t* d_words, int64_t n_rows, int64_t n_cols, void* stream);

/* Tuning knobs (process-wide): "cta_group" (2 = 256x256 tiles on an SM pair,
 * 1 = 128x128 on one SM), "prefetch" (L2 prefetch distance in k-blocks),
 * "l2_hint" (0 normal, 1 evict_last, 2 evict_first, 3 / 4 row blocks evict_last +
 * column blocks evict_first / normal), "band" (tile rows per
 * band of the tile order), "stages" (smem ring depth), "epi_warps" (8 or 16
 * epilogue warps), "fixed" (exact-mode epilogue: 1 adaptive per tile, default;
 * 0 FP64 only; 2 fixed-point table only; 3 hybrid only), "table_thr" (adaptive threshold on
 * the tile's column-sum spread), "pace" (L2 pacing window in k-blocks that
 * keeps the SM pairs' K sweeps together: -1 auto (default), 0 off), "tail"
 * (the last partial round of tiles split over the idle SM pairs: 1 auto,
 * default; 0 off; 2 column slices; 3 K ranges), "fp4" (1 = e2m1 operands on
 * kind::mxf4 when N < 2^24, default; 0 = int8), "evac" (e2m1: evacuate the
 * accumulator before FP64-free epilogues; 1 default, 0 off, 2 always),
 * "shard" (8 ranks: 1 = column-group pairs, default; 0 = round robin),
 * "hybrid" (exact-mode tiles off the table path: 0 = FP64, default; 1 = three
 * table gathers + T(c00) computed -- slower on every config measured),
 * "unperm_ctas" (CTAs per SM of mi_unpermute: 0 = auto by row width, default; 1..4), "ingest"
 * (mi_all_pairs_host: S = 1..16 column groups uploaded, unpacked, computed and
 * copied back in a pipeline, default 4; 0 = one upload, row-band egress),
 * "ingest_split" (0 = even group sizes, default; 1 = doubling), "serp" (1 =
 * odd tile rounds sweep K backwards for L2 reuse across rounds, default; 0 = always forwards),
 * "f32_epi" (float32 output, exact mode: tiles off the table path run the
 * FP32-pipe epilogue beside the next tile's MMAs; 1 default, 0 = FP64), "xp"
 * (the word-operand build of mi_all_pairs_host and the Python engine: -1 auto
 * = when m_pad <= "xp_cols", default 3072 (a third of it for an odd word count
 * per column, which needs a padded copy); 0 never; 1 whenever the operands
 * are e2m1), "xp_diag_w" (word-operand build: cost of a diagonal tile in
 * percent of an off-diagonal one, 10..100, which weights the K-range units of
 * the last partial round; default 90).  Also settable as MI_B200_<KEY> env vars. */
int mi_set_tuning(const char* key, int value);
int mi_get_tuning(const char* key); /* -1 for an unknown key (and for "pace" = auto) */
/* release the cached device workspaces of mi_*_host */
void mi_release_workspace(void);

/* Measured tensor peak of this device (the roofline denominator of the fused
 * kernel): every SM pair issues tcgen05.mma.cta_group::2 M=256 N=256 back to
 * back on shared-memory-resident operands -- kind::mxf4 with unit scales
 * (fp4 = 1, the fused kernel's instruction below 2^24 rows) or kind::i8
 * (fp4 = 0) -- for about `seconds` (short = burst clocks, >= 1 s = sustained
 * under the power cap).  Outputs (any may be NULL): dense tensor ops/s (2 per
 * MAC), MACs per clock per SM, and the effective SM clock in MHz. */
int mi_tensor_peak(int device, int fp4, double seconds, double* ops_per_s, double* macs_per_clk_sm,
                   double* sm_mhz);

#ifdef __cplusplus
}
#endif
#endif /* MIMATRIX_B200_H */
