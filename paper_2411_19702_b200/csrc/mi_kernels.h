// Internal (C++) interface between the C-ABI layer (capi.cu) and the kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#define MI_OUT_COUNTS 0
#define MI_OUT_F64 1
#define MI_OUT_F32 2
#define MI_MODE_EXACT 0
#define MI_MODE_EPSILON 1


namespace mib200 {

struct ColStat;

constexpr int kTailMaxUnits = 148;      // split tail units (<= clusters): flag pairs and partial slots
constexpr int kTailSumDepth = 4;        // K-range tail: other units' partials loaded per step of the sum

struct GramMiParams {
    const ColStat* colstat; // [m_pad] per-column marginals (kernel 1)
    const int2* tiles;      // [n_tiles] (I, J) tile coordinates, I <= J
    int n_tiles;
    int num_k_blocks;       // N_pad / 128
    int n_rows;             // N
    int m;                  // real columns (outputs beyond m are not written)
    int64_t ld_out;         // output row pitch in elements (0: packed upper triangle)
    int tile_major;         // 1: tile t of the list is stored at out + t TS^2 (TS x TS, row pitch TS),
                            // no mirror (the sharded form; mi_scatter_tiles places tiles + mirrors)
    void* out;              // int32 / double / float, row-major m x ld_out
    double eps;
    int include_diagonal;
    int prefetch_dist;      // k-blocks of L2 prefetch ahead of the TMA ring (0 = off)
    int l2_hint;            // operand loads: 0 normal, 1 evict_last, 2 evict_first, 3 / 4 rows evict_last + columns evict_first / normal
    int debug;              // experiments only (bit mask): 1 = compute but skip the output stores,
                            // 2 = skip the mirror stores, 4 = skip the direct stores, 8 = L2
                            // evict_first hint on the output stores, 16 = no MMAs (data movement only);
                            // word-operand build: 32 = no expansion, 64 = no word loads
    long long* trace;       // experiments only: per-tile timestamps of cluster 0 (or nullptr); word-operand
                            // build: per-phase cycle sums of cluster 0's expanders at [2048, 2080)
    unsigned long long rcp; // fixed point: round(2^(62 + nb) / N), nb = bit length of N
    int off0;               // fixed point: -(nb - 2) - s
    int fix_s;              // fixed point: scale s of the c log2 c terms
    const long long* xlogx; // exact mode: fixed-point T(c) = c log2(c) 2^s, c = 0..N (or nullptr)
    const int2* blkrange;   // exact mode: (min, max) column sum per 128-column block
    int table_thr;          // table path when the tile's two column-sum ranges sum to <= this
    int hybrid;             // other exact-mode tiles: 1 = hybrid (3 table gathers + T(c00) computed), 0 = FP64
    int f32_epi;            // float32 output, exact mode: tiles off the table path run the FP32-pipe
                            // epilogue (f32_mi, milog.cuh) instead of FP64, evacuated like the table path
    const float* fix_r;     // fix_xlog2x mantissa tables in global memory (hybrid path)
    const float2* fix_lg;
    unsigned int* row_done; // optional: per tile row I, +1 per CTA when its part of tile (I, J) is
                            // stored (system scope; lets the host stream finished rows to host)
    unsigned int* pace;     // optional: per-cluster k-block progress, stride kPaceStride (L2 pacing)
    int pace_window;        // leader producers stay within this many k-blocks of the slowest pair (0 = off)
    // Tail split of the last, partial round: tiles [0, n_full) are dealt
    // whole, round robin; tail tile i = t - n_full becomes s_i = tail_cnt[i]
    // units, run by consecutive clusters u = u0_i + c (u0_i = the counts
    // before it; tail_units = their sum):
    //  tail_kmode 0 (short K): unit c = column slice [c W, (c + 1) W) of the
    //    tile with the full K range, W = TS / s_i (all s_i = tail_split) --
    //    no partial sums;
    //  tail_kmode 1 (long K; a narrow slice would be load-bound): unit c = K
    //    range c of s_i of the full tile (s_i may differ per tile: weighted by
    //    tile cost).  Every unit stores its int32 accumulator in tail_part
    //    (slot u, 128 x TS per CTA) and bumps tail_flag[i * 2 + rank] (zeroed
    //    by the host before the launch); units c < tail_epi (<= every s_i)
    //    then wait for all s_i partials and run the epilogue of column slice c
    //    (TS / tail_epi wide) on their sum.
    int tail_units;
    unsigned char tail_cnt[kTailMaxUnits];
    int serp;               // 1: odd tile rounds sweep K backwards (L2 reuse across rounds)
    int evac;               // fp4: evacuate the accumulator before the epilogue (0 off, 1 FP64-free
                            // epilogues, 2 always)
    int n_full;
    int tail_split;         // 1 = no split, else the largest tail_cnt
    int tail_kmode;
    int tail_epi;
    unsigned int* tail_flag;
    uint32_t* tail_part;
    // Word-operand build (XP): the operands are expanded from the packed words
    // (m, nw) by producer warps straight into the swizzled shared-memory
    // stages; X never exists in HBM (tall-N / narrow-m shapes).
    const uint64_t* words;
    int64_t nw;
    // XP statistics mode (the tall-N step in one launch; all-tail K-range
    // schedules with every tile): the expanders count the ones of each column
    // on the diagonal tiles' units (they read every word of those columns
    // exactly once) into colstat[c].vi, and the epilogue warps -- idle until
    // the units finish -- build the T table, wait for the counts, write the
    // column statistics and meet at a grid-wide barrier before any epilogue.
    int xp_stats;
    unsigned int* xp_sync;        // [0] diagonal expander-warp completions, [1] CTAs done (zeroed by the host)
    ColStat* colstat_w;           // writable alias of colstat
    int32_t* colsum;              // optional column-sum output
    int2* blkrange_w;             // writable alias of blkrange
    long long* xlogx_w;           // the T table to build (or nullptr: none)
};
constexpr int kXpRowWarps = 4;          // word-operand build: warps covering one 128-row operand half
constexpr int kXpWarps = 2 * kXpRowWarps;  // word-operand build: expander warps per CTA (two groups)
constexpr int kXpEpiWarps = 4;          // word-operand build: epilogue warps
constexpr int kXpStages = 4;            // word-operand build: operand ring depth (a raw-word ring sits in front)
constexpr int kPaceStride = 8;          // u32 per cluster slot (one 32-B sector each)
constexpr int kPaceMaxClusters = 256;
constexpr long long kXlogxMaxN = 1ll << 24;  // table path: N < 2^24 (8 (N + 1) bytes)
constexpr int kFixLogBitsH = 10;             // = kFixLogBits (fixlog_table.h), for host code
constexpr long long kFixTabBytes = (1ll << kFixLogBitsH) * 12;  // kFixR floats + kFixLG float2s
constexpr long long kFp4MaxN = 1ll << 24;    // e2m1 operands: fp32 accumulators exact below 2^24

// fp4: operand X holds e2m1 nibbles (kind::mxf4 build, cg == 2 only), else int8 bytes
cudaError_t launch_gram_mi(int cg, bool fp4, int out_kind, int mode, int stages, int epi_warps,
                           const CUtensorMap& tmap, const GramMiParams& p, int num_sms, cudaStream_t stream);
// The word-operand build (p.words, p.nw; e2m1 operands expanded in the
// producer, CTA pairs, 4 epilogue warps, unpaced).
// tmap: the words (m, nw) uint64 as a 2-D tensor, 16 x 128 boxes, 128-byte swizzle
cudaError_t launch_gram_mi_words(int out_kind, int mode, const CUtensorMap& tmap, const GramMiParams& p, int num_sms,
                                 cudaStream_t stream);
int gram_mi_tile_size(int cg);

// block_mask (device, one byte per tile-size column block, or nullptr = all):
// expand only the marked blocks of X (a rank's share); fp4: write X as e2m1 nibbles (2 rows per byte, ld = bytes per column row
// band = N_pad / 2), else int8 bytes (ld = N_pad)
cudaError_t launch_unpack_colsum(const uint64_t* words, int64_t n_rows, int64_t m, int64_t nw,
                                 int8_t* x, int64_t ld, int64_t m_pad, int32_t* colsum,
                                 ColStat* colstat, long long* xlogx, int2* blkrange, float* fixr, bool fp4,
                                 const uint8_t* block_mask, int tile, int num_sms, cudaStream_t stream,
                                 const int32_t* perm = nullptr);

// The same in pieces, for staged ingest: the prologue (per-column counters,
// block ranges, the fixed-point table) once, then the expansion + column
// statistics of columns [c_begin, c_end) (c_begin a multiple of 32, c_end <=
// m_pad) as their words arrive.  blkrange = nullptr when there is no table.
// table = false: everything but the T table (the word-operand statistics mode builds it in the fused launch)
cudaError_t launch_unpack_prep(int64_t n_rows, int64_t m_pad, ColStat* colstat, long long* xlogx, int2* blkrange,
                               float* fixr, int num_sms, cudaStream_t stream, bool table = true);
cudaError_t launch_unpack_range(const uint64_t* words, int64_t n_rows, int64_t m, int64_t nw, int8_t* x, int64_t ld,
                                int64_t m_pad, int32_t* colsum, ColStat* colstat, int2* blkrange, bool fp4,
                                const uint8_t* block_mask, int tile, int64_t c_begin, int64_t c_end, int num_sms,
                                cudaStream_t stream, const int32_t* perm = nullptr);

// Device packing (pack.cu): row-major uint8 0/1 bits (n_rows x m, row pitch
// ld bytes) -> words (m, ceil(n_rows / 64)) uint64; *bad |= 1 on a byte > 1.
cudaError_t launch_pack_bits(const uint8_t* bits, int64_t n_rows, int64_t m, int64_t ld, uint64_t* words, int* bad,
                             cudaStream_t stream);

// binmat.to_dense on the device (pack.cu): CSC row indices (indptr[m + 1]) ->
// words (zeroed first); *bad |= 1 on an index outside [0, n_rows).
cudaError_t launch_pack_sparse(const int64_t* indices, const int64_t* indptr, int64_t n_rows, int64_t m,
                               uint64_t* words, int* bad, int num_sms, cudaStream_t stream);

// words (m, nw) -> the same with row pitch `pitch` words (pack.cu)
cudaError_t launch_pitch_words(const uint64_t* src, int64_t nw, uint64_t* dst, int64_t pitch, int64_t m, int num_sms,
                               cudaStream_t stream);

// Column order by column sum (order.cu): perm[s] = column in operand slot s
// (ascending sum, ties by column index), inv[perm[s]] = s; spread (device
// int[2], or nullptr) = (min, max) column sum.
cudaError_t launch_column_order(const uint64_t* words, int64_t n_rows, int64_t m, int32_t* perm, int32_t* inv,
                                int* spread, int num_sms, cudaStream_t stream);
// out[r][c] = in[inv[r]][inv[c]] for r, c < m; esz 4 or 8 bytes
cudaError_t launch_unpermute(const void* in, int64_t ld_in, void* out, int64_t ld_out, int64_t m, int esz,
                             const int32_t* inv, int num_sms, int smem_bytes, int ctas_per_sm, cudaStream_t stream);

// Sharded-result gather (scatter.cu): tile-major shards (ts x ts per tile, tile k
// of `tiles` at src + k ts^2) -> rows/columns of a full matrix (device or mapped
// host memory), plus the transposed mirror of off-diagonal tiles.
cudaError_t launch_scatter_tiles(const void* src, const int32_t* tiles, int64_t n_tiles, int ts, int64_t m, int esz,
                                 void* dst, int64_t ld, bool mirror, cudaStream_t stream);

// Tensor-peak probe (probe.cu): reps x 16 back-to-back 2-SM MMAs per SM pair;
// d_cycles[pair] = clock64 cycles of the issuing thread.
cudaError_t launch_tensor_peak(bool fp4, int reps, int num_sms, long long* d_cycles, cudaStream_t stream);
double tensor_peak_macs_per_pair(bool fp4, int reps);

cudaError_t launch_generate_words(uint64_t* words, int64_t n_rows, int64_t m, uint64_t seed,
                                  const uint64_t* col_threshold, const uint8_t* col_kind,
                                  const int32_t* col_src, uint64_t flip_threshold,
                                  uint64_t flip_seed, cudaStream_t stream);

}  // namespace mib200
