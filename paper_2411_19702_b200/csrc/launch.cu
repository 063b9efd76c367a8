// C-ABI entry points over device pointers: kernel 1 (unpack + column
// statistics), the fused Gram + MI kernel (launch_fused: tile list, tail
// split, L2 pacing, TMA descriptor), packing, column order, the generator
// and the tensor-peak probe.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <chrono>
#include <mutex>
#include <thread>
#include <condition_variable>
#include <vector>

#include "../../include/mimatrix_b200.h"
#include "capi_internal.h"
#include "mi_kernels.h"
#include "milog.cuh"

using namespace mib200;
using namespace mib200::capi;

namespace mib200 {
namespace capi {

long long* g_trace = nullptr;  // experiments only (mi_debug_set_trace)

// Per-device pacing slots of the fused kernel (kPaceMaxClusters x 32 B),
// allocated once and initialised to "finished" (0xFF bytes).
std::mutex g_pace_mu;
unsigned int* g_pace[64] = {};

// L2 pacing window in k-blocks (tuning "pace": -1 auto, 0 off, > 0 window).
// Auto paces long runs -- many tile rounds or long K -- where the pairs drift
// apart and the L2 stops sharing their operand reads (r01 sweep:
// config 5 175 -> 108 ms, config 4 45.5 -> 40.3 ms); short runs (config 3,
// 12 rounds) only pay the waits.
int pace_window(int64_t n_tiles, int nkb, int num_sms) {
    const int t = tuning().pace;
    if (t >= 0) return t;
    const int clusters = num_sms / 2;
    const int64_t rounds = (n_tiles + clusters - 1) / clusters;
    return (rounds > 16 || nkb > 2048) ? 32 : 0;
}

// Tail split of the last partial round (GramMiParams::tail_*): its r tiles
// become units so that the clusters share it instead of r of them.
// Short K (< kTailKMinKb k-blocks; latency-bound): column slices of the tile
// with the full K range, s a power of two, slices >= 32 wide.  Long K (the
// slices would be load-bound: a narrow MMA still streams a full A block):
// K ranges of the full tile, every cluster used: tile i gets s_i units, dealt
// one at a time to the tile whose units would run longest (w_i / s_i, w_i its
// cost weight; equal weights give counts that differ by at most one), and
// the int32 partials of a tile are summed by e <= min s_i epilogue units, one
// column slice each, at least 16 columns per epilogue warp (epi_parts warps
// share a TMEM lane quadrant; config 3: 820 tiles = 11 rounds of 74 + 6; the
// 6 run as 74 K ranges, summed by 8 epilogue slices each).  Weights: `h_tiles` (the
// host copy of the launch's tile list, or nullptr) marks the diagonal tail
// tiles, which cost diag_w percent of an off-diagonal one (the word-operand
// build stages one operand copy for them; knob "xp_diag_w").
// Knob "tail": 0 off, 1 auto, 2 slices only, 3 K ranges only.
constexpr int kTailKMinKb = 256;
int tail_epi_parts(bool xp) { return (xp ? kXpEpiWarps : tuning().epi_warps) / 4; }
TailPlan tail_plan(int64_t n_tiles, int cg, int clusters, int nkb, const int32_t* h_tiles, int diag_w, int epi_parts) {
    TailPlan tp{};
    tp.n_full = (int)n_tiles;
    tp.split = 1;
    tp.kmode = 0;
    tp.epi = 1;
    tp.units = 0;
    const int mode = tuning().tail;
    if (!mode || clusters < 2) return tp;
    const int64_t r = n_tiles % clusters;
    if (r == 0 || r > kTailMaxUnits) return tp;
    const bool kmode = mode == 3 || (mode == 1 && nkb >= kTailKMinKb);
    int s = 1, e = 1;
    while (e * 2 * 32 <= 128 * cg && r * e * 2 <= clusters) e *= 2;  // power-of-two column slices
    if (kmode) {  // epilogue slices: 16 columns per epilogue warp column part at least
        e = 1;
        while (e * 2 * 16 * epi_parts <= 128 * cg) e *= 2;
    }
    const int cap = std::min(std::min(nkb, kTailMaxUnits), 255);
    if (kmode) {
        if (clusters / r < 2 || cap < 2) return tp;
        const int budget = std::min(clusters, kTailMaxUnits);
        int w[kTailMaxUnits];
        int used = 0;
        for (int i = 0; i < (int)r; ++i) {
            const int64_t t = n_tiles - r + i;
            const bool diag = h_tiles && h_tiles[2 * t] == h_tiles[2 * t + 1];
            w[i] = diag ? std::max(1, std::min(diag_w, 100)) : 100;
            tp.cnt[i] = 2;
            used += 2;
        }
        for (; used < budget; ++used) {  // the next unit to the tile whose units run longest
            int best = -1;
            for (int i = 0; i < (int)r; ++i)
                if (tp.cnt[i] < cap && (best < 0 || (int64_t)w[i] * tp.cnt[best] > (int64_t)w[best] * tp.cnt[i]))
                    best = i;
            if (best < 0) break;
            ++tp.cnt[best];
        }
        s = 2;
        int smin = cap;
        for (int i = 0; i < (int)r; ++i) {
            s = std::max(s, (int)tp.cnt[i]);
            smin = std::min(smin, (int)tp.cnt[i]);
        }
        while (e > smin) e /= 2;  // epilogue slices stay a power of two
        tp.units = used;
    } else {
        s = e;
        if (s < 2 || r * s > kTailMaxUnits) return tp;
        for (int i = 0; i < (int)r; ++i) tp.cnt[i] = (unsigned char)s;
        tp.units = (int)(r * s);
    }
    tp.n_full = (int)(n_tiles - r);
    tp.split = s;
    tp.kmode = kmode ? 1 : 0;
    tp.epi = kmode ? e : s;
    return tp;
}

std::mutex g_tail_mu;
unsigned int* g_tail_flag[64] = {};
uint32_t* g_tail_part[64] = {};
cudaEvent_t g_tail_ev[64] = {};  // completion of the last launch that used the slots

int tail_slots(int device, unsigned int** flag, uint32_t** part) {
    std::lock_guard<std::mutex> lk(g_tail_mu);
    if (!g_tail_flag[device]) {
        MI_CUDA(cudaEventCreateWithFlags(&g_tail_ev[device], cudaEventDisableTiming));
        unsigned int* f = nullptr;
        uint32_t* q = nullptr;
        MI_CUDA(cudaMalloc((void**)&f, (size_t)kTailMaxUnits * 2 * 4));
        MI_CUDA(cudaMalloc((void**)&q, (size_t)kTailMaxUnits * 128 * 256 * 4));
        g_tail_flag[device] = f;
        g_tail_part[device] = q;
    }
    *flag = g_tail_flag[device];
    *part = g_tail_part[device];
    return MI_OK;
}

std::mutex g_xp_mu;
unsigned int* g_xp_sync[64] = {};
int xp_sync_slots(int device, unsigned int** out) {
    std::lock_guard<std::mutex> lk(g_xp_mu);
    if (!g_xp_sync[device]) MI_CUDA(cudaMalloc((void**)&g_xp_sync[device], 64));
    *out = g_xp_sync[device];
    return MI_OK;
}

int pace_slots(int device, unsigned int** out) {
    std::lock_guard<std::mutex> lk(g_pace_mu);
    if (!g_pace[device]) {
        const size_t bytes = (size_t)kPaceMaxClusters * kPaceStride * 4;
        unsigned int* p = nullptr;
        MI_CUDA(cudaMalloc((void**)&p, bytes));
        MI_CUDA(cudaMemset(p, 0xFF, bytes));
        MI_CUDA(cudaDeviceSynchronize());
        g_pace[device] = p;
    }
    *out = g_pace[device];
    return MI_OK;
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

int get_encode(PFN_cuTensorMapEncodeTiled_v12000* fn) {
    std::call_once(g_encode_once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!g_encode) return fail(MI_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    *fn = g_encode;
    return MI_OK;
}

// k-blocked K-major int8 operand X ([ld/128][m_pad][128] bytes) as a 3-D TMA
// tensor: 128-byte x 128-row boxes (one contiguous 16 KB chunk each), 128B
// swizzle (matches the UMMA descriptors).
int make_tmap(CUtensorMap* tm, const int8_t* x, int64_t ld, int64_t m_pad) {
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    int rc = get_encode(&enc);
    if (rc) return rc;
    cuuint64_t gdim[3] = {128, (cuuint64_t)m_pad, (cuuint64_t)(ld / 128)};
    cuuint64_t gstride[2] = {128, (cuuint64_t)m_pad * 128};
    cuuint32_t box[3] = {128, 128, 1};
    cuuint32_t estride[3] = {1, 1, 1};
    CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(x), gdim, gstride, box,
                     estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(MI_ERR_CUDA, "cuTensorMapEncodeTiled failed (CUresult %d)", (int)r);
    return MI_OK;
}

// The packed words (m, nw) uint64 as a 2-D TMA tensor for the word-operand
// build: 16-word (4 k-block, 128-byte) x 128-column boxes, 128-byte swizzle,
// zero fill beyond nw and m.  The row pitch (words) must be even: a multiple
// of 16 bytes.
int make_tmap_words(CUtensorMap* tm, const uint64_t* words, int64_t nw, int64_t pitch, int64_t m) {
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    int rc = get_encode(&enc);
    if (rc) return rc;
    cuuint64_t gdim[2] = {(cuuint64_t)nw, (cuuint64_t)m};
    cuuint64_t gstride[1] = {(cuuint64_t)pitch * 8};
    cuuint32_t box[2] = {16, 128};
    cuuint32_t estride[2] = {1, 1};
    CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<uint64_t*>(words), gdim, gstride, box, estride,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(MI_ERR_CUDA, "cuTensorMapEncodeTiled (words) failed (CUresult %d)", (int)r);
    return MI_OK;
}

// rcp = round(2^(62 + nb) / N) and off0 = -(nb - 2) - s for fixed_to_fp
void fixed_point_consts(int64_t N, unsigned long long* rcp, int* off0) {
    int nb = 0;
    while (nb < 63 && (1ll << nb) <= N) ++nb;
    const unsigned __int128 num = (unsigned __int128)1 << (62 + nb);
    *rcp = (unsigned long long)((num + (unsigned __int128)(N / 2)) / (unsigned __int128)N);
    *off0 = -(nb - 2) - xlogx_scale(N);
}

}  // namespace capi
}  // namespace mib200

extern "C" {

int mi_unpack_colsum(const uint64_t* d_words, int64_t n_rows, int64_t n_cols, int8_t* d_kmajor, int64_t ld,
                     void* d_colstat, int32_t* d_colsum, void* stream) {
    return mi_unpack_colsum_blocks(d_words, n_rows, n_cols, d_kmajor, ld, d_colstat, d_colsum, nullptr, stream);
}

int mi_unpack_colsum_blocks(const uint64_t* d_words, int64_t n_rows, int64_t n_cols, int8_t* d_kmajor, int64_t ld,
                            void* d_colstat, int32_t* d_colsum, const uint8_t* d_block_mask, void* stream) {
    int rc = check_shape(n_rows, n_cols);
    if (rc) return rc;
    if (ld < mi_kmajor_ld(n_rows) || ld % 128)
        return fail(MI_ERR_DIMENSION, "ld %lld must be a multiple of 128 and >= %lld", (long long)ld,
                    (long long)mi_kmajor_ld(n_rows));
    DevInfo info;
    if ((rc = current_device_info(&info))) return rc;
    const int64_t nw = (n_rows + 63) / 64;
    if (!d_colstat) return fail(MI_ERR_DOMAIN, "d_colstat is required");
    MI_CUDA(launch_unpack_colsum(d_words, n_rows, n_cols, nw, d_kmajor, ld, mi_kmajor_rows(n_cols), d_colsum,
                                 (ColStat*)d_colstat, xlogx_ptr(d_colstat, n_rows, n_cols),
                                 blkrange_ptr(d_colstat, n_rows, n_cols), fixr_ptr(d_colstat, n_rows, n_cols),
                                 operand_fp4(n_rows), d_block_mask,
                                 mi_tile_size(), info.num_sms, (cudaStream_t)stream));
    return MI_OK;
}

int mi_unpack_prep(int64_t n_rows, int64_t n_cols, void* d_colstat, void* stream) {
    int rc = check_shape(n_rows, n_cols);
    if (rc) return rc;
    if (!d_colstat) return fail(MI_ERR_DOMAIN, "d_colstat is required");
    DevInfo info;
    if ((rc = current_device_info(&info))) return rc;
    MI_CUDA(launch_unpack_prep(n_rows, mi_kmajor_rows(n_cols), (ColStat*)d_colstat,
                               xlogx_ptr(d_colstat, n_rows, n_cols), blkrange_ptr(d_colstat, n_rows, n_cols),
                               fixr_ptr(d_colstat, n_rows, n_cols), info.num_sms, (cudaStream_t)stream));
    return MI_OK;
}

int mi_unpack_colsum_range(const uint64_t* d_words, int64_t n_rows, int64_t n_cols, int8_t* d_kmajor, int64_t ld,
                           void* d_colstat, int32_t* d_colsum, const uint8_t* d_block_mask, int64_t c_begin,
                           int64_t c_end, void* stream) {
    int rc = check_shape(n_rows, n_cols);
    if (rc) return rc;
    if (ld < mi_kmajor_ld(n_rows) || ld % 128)
        return fail(MI_ERR_DIMENSION, "ld %lld must be a multiple of 128 and >= %lld", (long long)ld,
                    (long long)mi_kmajor_ld(n_rows));
    if (!d_colstat) return fail(MI_ERR_DOMAIN, "d_colstat is required");
    const int64_t m_pad = mi_kmajor_rows(n_cols);
    // both ends on multiples of 32: colstat_kernel's per-warp min/max reductions
    // need every lane of the range's last warp (m_pad is a multiple of 256, so
    // the last range can always end there)
    if (c_begin < 0 || c_begin % 32 || c_end % 32 || c_end > m_pad || c_begin >= c_end)
        return fail(MI_ERR_DIMENSION,
                    "column range [%lld, %lld) must start and end on multiples of 32 and lie in [0, %lld]",
                    (long long)c_begin, (long long)c_end, (long long)m_pad);
    DevInfo info;
    if ((rc = current_device_info(&info))) return rc;
    const int64_t nw = (n_rows + 63) / 64;
    long long* xl = xlogx_ptr(d_colstat, n_rows, n_cols);
    MI_CUDA(launch_unpack_range(d_words, n_rows, n_cols, nw, d_kmajor, ld, m_pad, d_colsum, (ColStat*)d_colstat,
                                xl ? blkrange_ptr(d_colstat, n_rows, n_cols) : nullptr, operand_fp4(n_rows),
                                d_block_mask, mi_tile_size(), c_begin, c_end, info.num_sms, (cudaStream_t)stream));
    return MI_OK;
}

int mi_gram_mi(const int8_t* d_kmajor, const void* d_colstat, int64_t n_rows, int64_t n_cols, int64_t ld,
               int mode, double epsilon, int include_diagonal, int out_kind, void* d_out, int64_t ld_out,
               const int32_t* d_tiles, int64_t n_tiles, void* stream) {
    return launch_fused(d_kmajor, d_colstat, n_rows, n_cols, ld, mode, epsilon, include_diagonal, out_kind, d_out,
                        ld_out, d_tiles, n_tiles, nullptr, (cudaStream_t)stream);
}

int mi_gram_mi_words(const uint64_t* d_words, const void* d_colstat, int64_t n_rows, int64_t n_cols, int mode,
                     double epsilon, int include_diagonal, int out_kind, void* d_out, int64_t ld_out,
                     const int32_t* d_tiles, int64_t n_tiles, void* stream) {
    if (!d_words || !d_colstat) return fail(MI_ERR_DOMAIN, "d_words and d_colstat are required");
    return launch_fused(nullptr, d_colstat, n_rows, n_cols, 0, mode, epsilon, include_diagonal, out_kind, d_out, ld_out,
                        d_tiles, n_tiles, nullptr, (cudaStream_t)stream, d_words);
}

int mi_gram_mi_words_stats(const uint64_t* d_words, void* d_colstat, int32_t* d_colsum, int64_t n_rows,
                           int64_t n_cols, int mode, double epsilon, int include_diagonal, int out_kind, void* d_out,
                           int64_t ld_out, const int32_t* d_tiles, int64_t n_tiles, void* stream) {
    if (!d_words || !d_colstat) return fail(MI_ERR_DOMAIN, "d_words and d_colstat are required");
    return launch_fused(nullptr, d_colstat, n_rows, n_cols, 0, mode, epsilon, include_diagonal, out_kind, d_out, ld_out,
                        d_tiles, n_tiles, nullptr, (cudaStream_t)stream, d_words, true, d_colsum);
}

int mi_colstat_words(const uint64_t* d_words, int64_t n_rows, int64_t n_cols, void* d_colstat, int32_t* d_colsum,
                     void* stream) {
    int rc = check_shape(n_rows, n_cols);
    if (rc) return rc;
    if (!d_words || !d_colstat) return fail(MI_ERR_DOMAIN, "d_words and d_colstat are required");
    DevInfo info;
    if ((rc = current_device_info(&info))) return rc;
    const int64_t nw = (n_rows + 63) / 64;
    // kernel 1 without the expansion (x = nullptr): column sums + statistics only
    MI_CUDA(launch_unpack_colsum(d_words, n_rows, n_cols, nw, nullptr, mi_kmajor_ld(n_rows), mi_kmajor_rows(n_cols),
                                 d_colsum, (ColStat*)d_colstat, xlogx_ptr(d_colstat, n_rows, n_cols),
                                 blkrange_ptr(d_colstat, n_rows, n_cols), fixr_ptr(d_colstat, n_rows, n_cols),
                                 operand_fp4(n_rows), nullptr, mi_tile_size(), info.num_sms, (cudaStream_t)stream));
    return MI_OK;
}

int mi_scatter_tiles(const void* d_src, const int32_t* d_tiles, int64_t n_tiles, int64_t n_cols, int esz, void* d_dst,
                     int64_t ld_dst, int mirror, void* stream) {
    if (n_cols < 1 || n_cols > 0x7FFFFFFF) return fail(MI_ERR_DIMENSION, "n_cols must be in [1, 2^31)");
    if (esz != 4 && esz != 8) return fail(MI_ERR_DOMAIN, "esz must be 4 or 8");
    if (ld_dst < n_cols) return fail(MI_ERR_DIMENSION, "ld_dst %lld < n_cols", (long long)ld_dst);
    if (n_tiles < 0 || n_tiles > 0x7FFFFFFF) return fail(MI_ERR_DIMENSION, "bad n_tiles");
    if (n_tiles == 0) return MI_OK;
    if (!d_src || !d_tiles || !d_dst) return fail(MI_ERR_DOMAIN, "d_src, d_tiles and d_dst are required");
    // pinned host destinations are written through their device alias
    void* dst = d_dst;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, d_dst) != cudaSuccess) {
        cudaGetLastError();
        return fail(MI_ERR_DOMAIN, "d_dst is neither device memory nor pinned host memory");
    }
    if (a.type == cudaMemoryTypeHost) {
        if (!a.devicePointer) return fail(MI_ERR_DOMAIN, "host d_dst is not mapped (register it with mi_host_register)");
        dst = a.devicePointer;
    } else if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) {
        return fail(MI_ERR_DOMAIN, "d_dst is pageable host memory: pin it (mi_host_register) first");
    }
    MI_CUDA(launch_scatter_tiles(d_src, d_tiles, n_tiles, mi_tile_size(), n_cols, esz, dst, ld_dst, mirror != 0,
                                 (cudaStream_t)stream));
    return MI_OK;
}

int mi_pack_bits(const uint8_t* d_bits, int64_t n_rows, int64_t n_cols, int64_t ld_bits, uint64_t* d_words,
                 int32_t* d_bad, void* stream) {
    int rc = check_shape(n_rows, n_cols);
    if (rc) return rc;
    if (ld_bits < n_cols) return fail(MI_ERR_DIMENSION, "ld_bits %lld < n_cols", (long long)ld_bits);
    if (!d_bits || !d_words || !d_bad) return fail(MI_ERR_DOMAIN, "d_bits, d_words and d_bad are required");
    MI_CUDA(launch_pack_bits(d_bits, n_rows, n_cols, ld_bits, d_words, reinterpret_cast<int*>(d_bad),
                             (cudaStream_t)stream));
    return MI_OK;
}

int mi_pack_sparse(const int64_t* d_indices, const int64_t* d_indptr, int64_t n_rows, int64_t n_cols,
                   uint64_t* d_words, int32_t* d_bad, void* stream) {
    int rc = check_shape(n_rows, n_cols);
    if (rc) return rc;
    if (!d_indptr || !d_words || !d_bad) return fail(MI_ERR_DOMAIN, "d_indptr, d_words and d_bad are required");
    DevInfo info;
    if ((rc = current_device_info(&info))) return rc;
    MI_CUDA(launch_pack_sparse(d_indices, d_indptr, n_rows, n_cols, d_words, reinterpret_cast<int*>(d_bad),
                               info.num_sms, (cudaStream_t)stream));
    return MI_OK;
}

int mi_column_order(const uint64_t* d_words, int64_t n_rows, int64_t n_cols, int32_t* d_perm, int32_t* d_inv,
                    int32_t* d_spread, void* stream) {
    int rc = check_shape(n_rows, n_cols);
    if (rc) return rc;
    if (n_cols > 0x7FFFFFFF) return fail(MI_ERR_DIMENSION, "n_cols must fit in int32 for a column order");
    if (!d_words || !d_perm || !d_inv) return fail(MI_ERR_DOMAIN, "d_words, d_perm and d_inv are required");
    DevInfo info;
    if ((rc = current_device_info(&info))) return rc;
    MI_CUDA(launch_column_order(d_words, n_rows, n_cols, d_perm, d_inv, reinterpret_cast<int*>(d_spread),
                                info.num_sms, (cudaStream_t)stream));
    return MI_OK;
}

int mi_unpack_colsum_ordered(const uint64_t* d_words, int64_t n_rows, int64_t n_cols, const int32_t* d_perm,
                             int8_t* d_kmajor, int64_t ld, void* d_colstat, int32_t* d_colsum, void* stream) {
    int rc = check_shape(n_rows, n_cols);
    if (rc) return rc;
    if (ld < mi_kmajor_ld(n_rows) || ld % 128)
        return fail(MI_ERR_DIMENSION, "ld %lld must be a multiple of 128 and >= %lld", (long long)ld,
                    (long long)mi_kmajor_ld(n_rows));
    if (!d_colstat) return fail(MI_ERR_DOMAIN, "d_colstat is required");
    DevInfo info;
    if ((rc = current_device_info(&info))) return rc;
    const int64_t nw = (n_rows + 63) / 64;
    MI_CUDA(launch_unpack_colsum(d_words, n_rows, n_cols, nw, d_kmajor, ld, mi_kmajor_rows(n_cols), d_colsum,
                                 (ColStat*)d_colstat, xlogx_ptr(d_colstat, n_rows, n_cols),
                                 blkrange_ptr(d_colstat, n_rows, n_cols), fixr_ptr(d_colstat, n_rows, n_cols),
                                 operand_fp4(n_rows), nullptr, mi_tile_size(), info.num_sms, (cudaStream_t)stream,
                                 d_perm));
    return MI_OK;
}

int mi_unpermute(const void* d_in, int64_t ld_in, void* d_out, int64_t ld_out, int64_t n_cols, int esz,
                 const int32_t* d_inv, void* stream) {
    if (n_cols < 1 || n_cols > 0x7FFFFFFF) return fail(MI_ERR_DIMENSION, "n_cols must be in [1, 2^31)");
    if (esz != 4 && esz != 8) return fail(MI_ERR_DOMAIN, "esz must be 4 or 8");
    if (ld_in < n_cols || ld_out < n_cols) return fail(MI_ERR_DIMENSION, "ld_in and ld_out must be >= n_cols");
    if (!d_in || !d_out || !d_inv) return fail(MI_ERR_DOMAIN, "d_in, d_out and d_inv are required");
    if ((reinterpret_cast<uintptr_t>(d_in) | reinterpret_cast<uintptr_t>(d_out)) % (uintptr_t)esz)
        return fail(MI_ERR_DOMAIN, "d_in and d_out must be aligned to esz");
    const char* a0 = static_cast<const char*>(d_in);
    const char* b0 = static_cast<const char*>(d_out);
    const int64_t span_in = ((n_cols - 1) * ld_in + n_cols) * esz, span_out = ((n_cols - 1) * ld_out + n_cols) * esz;
    if (a0 < b0 + span_out && b0 < a0 + span_in) return fail(MI_ERR_DOMAIN, "d_in and d_out must not overlap");
    DevInfo info;
    int rc;
    if ((rc = current_device_info(&info))) return rc;
    int dev = 0, smem = 0;
    MI_CUDA(cudaGetDevice(&dev));
    MI_CUDA(cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    // CTAs per SM: the knob, or (0 = auto, default) as many whole source rows
    // as the SM's shared memory holds, up to 4, for rows up to 90 KB -- more
    // rows in flight per SM for narrower matrices (tools/unpermute_bench.py:
    // m = 5000 float64 0.125 -> 0.088 ms, m = 10000 float32 0.215 -> 0.174 ms),
    // one CTA for wider rows (m = 25000 float32 was slower with two).
    int ctas = tuning().unperm_ctas;
    if (ctas == 0) {
        const int64_t row = n_cols * esz + 1024;
        ctas = row > 90 * 1024 ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(4, (int64_t)smem / row));
    }
    int per_cta = smem / ctas - 1024;  // leave room for the per-CTA reserve
    per_cta = per_cta / 16 * 16;
    MI_CUDA(launch_unpermute(d_in, ld_in, d_out, ld_out, n_cols, esz, d_inv, info.num_sms, per_cta, ctas,
                             (cudaStream_t)stream));
    return MI_OK;
}

}  // extern "C"

int mib200::capi::launch_fused(const int8_t* d_kmajor, const void* d_colstat, int64_t n_rows, int64_t n_cols, int64_t ld, int mode,
                 double epsilon, int include_diagonal, int out_kind, void* d_out, int64_t ld_out, const int32_t* d_tiles,
                 int64_t n_tiles, unsigned int* row_done, cudaStream_t stream, const uint64_t* d_words, bool stats,
                 int32_t* d_colsum) {
    int rc = check_shape(n_rows, n_cols);
    if (rc) return rc;
    if ((rc = check_mode(mode, epsilon, out_kind))) return rc;
    // d_words: the word-operand build (expansion in the producer; no X, no TMA)
    const bool xp = d_words != nullptr;
    if (xp && !operand_fp4(n_rows))
        return fail(MI_ERR_DOMAIN, "the word-operand build needs e2m1 operands (n_rows < 2^24, SM-pair tiles)");
    if (!xp && (ld < mi_kmajor_ld(n_rows) || ld % 128))
        return fail(MI_ERR_DIMENSION, "ld %lld must be a multiple of 128 and >= %lld", (long long)ld,
                    (long long)mi_kmajor_ld(n_rows));
    if (ld_out != MI_PACKED_UPPER && ld_out != MI_TILE_MAJOR && ld_out < n_cols)
        return fail(MI_ERR_DIMENSION, "ld_out %lld < n_cols (or MI_PACKED_UPPER / MI_TILE_MAJOR)", (long long)ld_out);
    if (ld_out == MI_TILE_MAJOR && row_done)
        return fail(MI_ERR_DOMAIN, "row-band egress needs a full-matrix output");
    if (n_tiles < 0 || n_tiles > 0x7FFFFFFF) return fail(MI_ERR_DIMENSION, "bad n_tiles");
    if (n_tiles == 0) return MI_OK;
    if (out_kind == MI_OUT_COUNTS && mode != MI_MODE_EXACT)
        return fail(MI_ERR_DOMAIN, "counts export ignores the mode; pass MI_MODE_EXACT");
    if (xp && (reinterpret_cast<uintptr_t>(d_words) & 7) != 0) return fail(MI_ERR_DOMAIN, "words must be 8-byte aligned");
    if (!xp && (reinterpret_cast<uintptr_t>(d_kmajor) & 15) != 0)
        return fail(MI_ERR_DOMAIN, "kmajor operand must be 16-byte aligned");
    DevInfo info;
    if ((rc = current_device_info(&info))) return rc;
    CUtensorMap tm;
    if (!xp && (rc = make_tmap(&tm, d_kmajor, ld, mi_kmajor_rows(n_cols)))) return rc;
    // The words' TMA map needs a row pitch of a multiple of 16 bytes: an odd word
    // count per column (or a misaligned base) is first copied with one pad word
    // per column (stream-ordered scratch kept in the pool between calls; 0.5 GB
    // at N = 8e6, m = 512)
    const int64_t nw_x = (n_rows + 63) / 64;
    uint64_t* padded = nullptr;
    struct AsyncFree {  // released on the stream after whatever this call enqueued
        void** p;
        cudaStream_t s;
        ~AsyncFree() {
            if (*p) cudaFreeAsync(*p, s);
        }
    } padded_guard{(void**)&padded, stream};
    if (xp && ((nw_x & 1) || (reinterpret_cast<uintptr_t>(d_words) & 15))) {
        const int64_t pitch = nw_x + (nw_x & 1);
        const size_t bytes = (size_t)(n_cols * pitch * 8);
        cudaMemPool_t pool;
        int cur = 0;
        if (cudaGetDevice(&cur) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, cur) == cudaSuccess) {
            uint64_t keep = 0;
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            if (keep < bytes) {
                keep = bytes;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            }
        }
        MI_CUDA(cudaMallocAsync((void**)&padded, bytes, stream));
        MI_CUDA(launch_pitch_words(d_words, nw_x, padded, pitch, n_cols, info.num_sms, stream));
        if ((rc = make_tmap_words(&tm, padded, nw_x, pitch, n_cols))) return rc;
    } else if (xp && (rc = make_tmap_words(&tm, d_words, nw_x, nw_x, n_cols))) {
        return rc;
    }
    GramMiParams p;
    p.words = d_words;
    p.nw = (n_rows + 63) / 64;
    p.colstat = reinterpret_cast<const ColStat*>(d_colstat);
    p.tiles = reinterpret_cast<const int2*>(d_tiles);
    p.n_tiles = (int)n_tiles;
    p.num_k_blocks = (int)(mi_kmajor_ld(n_rows) / 128);
    p.n_rows = (int)n_rows;
    p.m = (int)n_cols;
    p.tile_major = ld_out == MI_TILE_MAJOR ? 1 : 0;
    p.ld_out = ld_out == MI_TILE_MAJOR ? (int64_t)mi_tile_size() : ld_out;
    p.out = d_out;
    p.eps = epsilon;
    p.include_diagonal = include_diagonal ? 1 : 0;
    p.prefetch_dist = prefetch_dist();
    p.l2_hint = l2_hint();
    p.debug = tuning().debug;
    p.row_done = row_done;
    p.trace = g_trace;
    int dev = 0;
    MI_CUDA(cudaGetDevice(&dev));
    p.evac = tuning().evac;
    p.serp = tuning().serp;
    p.pace = nullptr;
    p.pace_window = xp ? 0 : pace_window(n_tiles, p.num_k_blocks, info.num_sms);
    if (p.pace_window > 0 && (rc = pace_slots(dev, &p.pace))) return rc;
    // the diagonal tail tiles (cost weights of the K-range units): known for
    // the full list in the order the engine and the host paths build it (a
    // heuristic -- any order and any counts give the same results)
    std::vector<int32_t> canon;
    const int64_t T_side = tiles_per_side(n_cols);
    if (xp && n_tiles == T_side * (T_side + 1) / 2) canon = all_tiles(T_side, tile_band(), row_done ? 1 : 0);
    const TailPlan tp = tail_plan(n_tiles, cta_group(), info.num_sms / cta_group(), p.num_k_blocks,
                                  canon.empty() ? nullptr : canon.data(), xp ? tuning().xp_diag_w : 100,
                                  tail_epi_parts(xp));
    p.n_full = tp.n_full;
    p.tail_split = tp.split;
    p.tail_units = tp.units;
    memcpy(p.tail_cnt, tp.cnt, sizeof(p.tail_cnt));
    p.tail_kmode = tp.kmode;
    p.tail_epi = tp.epi;
    p.tail_flag = nullptr;
    p.tail_part = nullptr;
    // The K-range tail's flags and partial slots are one per device: launches
    // that use them are chained across streams (the next waits for the last)
    // so concurrent callers on different streams cannot mix their partials.
    std::unique_lock<std::mutex> tail_lk(g_tail_mu, std::defer_lock);
    if (tp.kmode) {
        if ((rc = tail_slots(dev, &p.tail_flag, &p.tail_part))) return rc;
        tail_lk.lock();
        MI_CUDA(cudaStreamWaitEvent(stream, g_tail_ev[dev], 0));
        MI_CUDA(cudaMemsetAsync(p.tail_flag, 0, (size_t)(n_tiles - tp.n_full) * 2 * 4, stream));
    }
    fixed_point_consts(n_rows, &p.rcp, &p.off0);
    p.fix_s = xlogx_scale(n_rows);
    p.xlogx = xlogx_ptr(const_cast<void*>(d_colstat), n_rows, n_cols);
    p.blkrange = blkrange_ptr(const_cast<void*>(d_colstat), n_rows, n_cols);
    p.fix_r = fixr_ptr(const_cast<void*>(d_colstat), n_rows, n_cols);
    p.fix_lg = p.fix_r ? reinterpret_cast<const float2*>(p.fix_r + (1 << kFixLogBitsH)) : nullptr;
    // exact-mode epilogue: 0 = FP64 only, 1 = adaptive per tile (default), 2 = table only
    p.table_thr = tuning().fixed == 0 ? -1 : tuning().fixed == 2 ? 0x7FFFFFFF : tuning().fixed == 3 ? -1 : tuning().table_thr;
    // tiles that miss the table threshold: hybrid (fixed 1 with hybrid on, or 3) or FP64
    p.hybrid = (tuning().fixed == 3 || (tuning().fixed == 1 && tuning().hybrid)) && p.fix_r ? 1 : 0;
    // float32 output: the FP32-pipe epilogue for those tiles (counts exact in fp32: N < 2^24)
    p.f32_epi = (tuning().f32_epi && tuning().fixed != 0 && out_kind == MI_OUT_F32 && n_rows < kFp4MaxN) ? 1 : 0;
    int eff_mode = out_kind == MI_OUT_COUNTS ? MI_MODE_EXACT : mode;
    // exact mode runs the FP64-free fixed-point epilogue whenever the table exists
    // stats: this call computes the column statistics too -- inside the launch
    // when every tile runs as K-range tail units (the expanders count the
    // diagonal units' columns), else by kernel 1's counting pass first
    p.xp_stats = 0;
    p.xp_sync = nullptr;
    p.colstat_w = reinterpret_cast<ColStat*>(const_cast<void*>(d_colstat));
    p.colsum = d_colsum;
    p.blkrange_w = blkrange_ptr(const_cast<void*>(d_colstat), n_rows, n_cols);
    p.xlogx_w = nullptr;
    if (stats) {
        ColStat* cs = reinterpret_cast<ColStat*>(const_cast<void*>(d_colstat));
        long long* xl = xlogx_ptr(const_cast<void*>(d_colstat), n_rows, n_cols);
        int2* br = blkrange_ptr(const_cast<void*>(d_colstat), n_rows, n_cols);
        float* fr = fixr_ptr(const_cast<void*>(d_colstat), n_rows, n_cols);
        const int64_t T = tiles_per_side(n_cols);
        const bool fused_stats = xp && n_tiles == T * (T + 1) / 2 && tp.n_full == 0 && tp.kmode && tp.split > 1 &&
                                 tuning().xp_stats;
        if (fused_stats) {
            if ((rc = xp_sync_slots(dev, &p.xp_sync))) return rc;
            MI_CUDA(launch_unpack_prep(n_rows, mi_kmajor_rows(n_cols), cs, xl, br, fr, info.num_sms, stream, false));
            MI_CUDA(cudaMemsetAsync(p.xp_sync, 0, 2 * sizeof(unsigned int), stream));
            p.xp_stats = 1;
            p.xlogx_w = xl;
        } else {
            MI_CUDA(launch_unpack_colsum(d_words, n_rows, n_cols, (n_rows + 63) / 64, xp ? nullptr : (int8_t*)d_kmajor,
                                         ld, mi_kmajor_rows(n_cols), d_colsum, cs, xl, br, fr, operand_fp4(n_rows),
                                         nullptr, mi_tile_size(), info.num_sms, stream));
        }
    }
    if (xp)
        MI_CUDA(launch_gram_mi_words(out_kind, eff_mode, tm, p, info.num_sms, stream));
    else
        MI_CUDA(launch_gram_mi(cta_group(), operand_fp4(n_rows), out_kind, eff_mode, tuning().stages,
                               tuning().epi_warps, tm, p, info.num_sms, stream));
    if (tp.kmode) MI_CUDA(cudaEventRecord(g_tail_ev[dev], stream));
    return MI_OK;
}

extern "C" {

int mi_generate_words(uint64_t* d_words, int64_t n_rows, int64_t n_cols, uint64_t seed,
                      const uint64_t* d_col_threshold, const uint8_t* d_col_kind, const int32_t* d_col_src,
                      uint64_t flip_threshold, uint64_t flip_seed, void* stream) {
    int rc = check_shape(n_rows, n_cols);
    if (rc) return rc;
    MI_CUDA(launch_generate_words(d_words, n_rows, n_cols, seed, d_col_threshold, d_col_kind, d_col_src,
                                  flip_threshold, flip_seed, (cudaStream_t)stream));
    return MI_OK;
}

// Not part of the public header: route per-tile timestamps of cluster 0 into a
// device buffer of 64 x 4 int64 (tools/trace_tiles.py) followed by 256 x 4
// per-cluster globaltimer stamps (start, main tiles done, tail done), or
// nullptr to stop.
void mi_debug_set_trace(void* d_buf) { g_trace = reinterpret_cast<long long*>(d_buf); }

int mi_tensor_peak(int device, int fp4, double seconds, double* ops_per_s, double* macs_per_clk_sm,
                   double* sm_mhz) {
    if (!(seconds > 0.0) || seconds > 60.0) return fail(MI_ERR_DOMAIN, "seconds must be in (0, 60]");
    DevInfo info;
    int rc = query_device(device, &info);
    if (rc) return rc;
    MI_CUDA(cudaSetDevice(device));
    const int pairs = info.num_sms / 2;
    long long* d_cyc = nullptr;
    MI_CUDA(cudaMalloc((void**)&d_cyc, (size_t)pairs * 8));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](int reps, float* ms) -> cudaError_t {
        cudaEventRecord(e0, 0);
        cudaError_t e = launch_tensor_peak(fp4 != 0, reps, info.num_sms, d_cyc, 0);
        if (e != cudaSuccess) return e;
        cudaEventRecord(e1, 0);
        if ((e = cudaEventSynchronize(e1)) != cudaSuccess) return e;
        return cudaEventElapsedTime(ms, e0, e1);
    };
    float ms = 0.f;
    int reps = 2000;
    cudaError_t e = run(reps, &ms);  // warm-up and calibration (~2 ms)
    if (e == cudaSuccess && ms > 0.f) {
        const double want = seconds * 1e3 / ms * reps;
        reps = (int)std::max(100.0, std::min(want, 2.0e9));
        e = run(reps, &ms);
    }
    std::vector<long long> cyc((size_t)pairs, 0);
    if (e == cudaSuccess) e = cudaMemcpy(cyc.data(), d_cyc, (size_t)pairs * 8, cudaMemcpyDeviceToHost);
    cudaFree(d_cyc);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (e != cudaSuccess) return cuda_fail(e, "tensor peak probe");
    long long mx = 1;
    for (long long c : cyc) mx = std::max(mx, c);
    const double macs_pair = tensor_peak_macs_per_pair(fp4 != 0, reps);
    if (ops_per_s) *ops_per_s = 2.0 * macs_pair * pairs / (ms * 1e-3);
    if (macs_per_clk_sm) *macs_per_clk_sm = macs_pair / (double)mx / 2.0;
    if (sm_mhz) *sm_mhz = (double)mx / (ms * 1e-3) / 1e6;
    return MI_OK;
}

}  // extern "C"
