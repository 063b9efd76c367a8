// C-ABI layer of libmimatrix_b200.so (declared in include/mimatrix_b200.h).
// Validation and error codes follow the reference's exception contract
// (errors.py:8-25, engine.py:36-44,157-158, binmat.py:71-80, gram.py:98-110).
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
#include "mi_kernels.h"
#include "milog.cuh"

using namespace mib200;

// fused kernel launch shared by mi_gram_mi and the host entry points (defined below)
int launch_fused(const int8_t* d_kmajor, const void* d_colstat, int64_t n_rows, int64_t n_cols, int64_t ld, int mode,
                 double epsilon, int include_diagonal, int out_kind, void* d_out, int64_t ld_out, const int32_t* d_tiles,
                 int64_t n_tiles, unsigned int* row_done, cudaStream_t stream);

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(MI_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

#define MI_CUDA(call)                                   \
    do {                                                \
        cudaError_t e_ = (call);                        \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

// Tuning knobs: defaults are the measured best; MI_B200_* env vars
// or mi_set_tuning() override them.  cta_group 2 = 256 x 256 tiles on a CTA
// pair (production); 1 = single-SM 128 x 128 tiles.
constexpr int kMaxIngestStages = 16;

int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return (e && *e) ? atoi(e) : dflt;
}
struct Tuning {
    int cta_group, prefetch, l2_hint, band, stages, epi_warps, debug, fixed, table_thr, pace, tail, fp4, evac, shard,
        hybrid, unperm_ctas, ingest, ingest_split, serp, f32_epi;
};
Tuning& tuning() {
    static Tuning t = {env_int("MI_B200_CTA_GROUP", 2) == 1 ? 1 : 2, env_int("MI_B200_PREFETCH", 0),
                       env_int("MI_B200_L2HINT", 1), env_int("MI_B200_BAND", 8),
                       env_int("MI_B200_STAGES", 6), env_int("MI_B200_EPI_WARPS", 8), env_int("MI_B200_DEBUG", 0),
                       env_int("MI_B200_FIXED", 1), env_int("MI_B200_TABLE_THR", 4096),
                       env_int("MI_B200_PACE", -1), env_int("MI_B200_TAIL", 1), env_int("MI_B200_FP4", 1),
                       env_int("MI_B200_EVAC", 1), env_int("MI_B200_SHARD", 1),
                       env_int("MI_B200_HYBRID", 0), env_int("MI_B200_UNPERM_CTAS", 0),
                       env_int("MI_B200_INGEST", 4), env_int("MI_B200_INGEST_SPLIT", 0),
                       env_int("MI_B200_SERP", 0), env_int("MI_B200_F32_EPI", 1)};
    return t;
}
int cta_group() { return tuning().cta_group; }
// Operand format: e2m1 nibbles for kind::mxf4 (twice the int8 MMA rate, half
// the bytes) on SM pairs while fp32 accumulation is exact (N < 2^24), else
// int8.  mi_unpack_colsum and mi_gram_mi both follow this rule, so the knob
// must not change between them.
bool operand_fp4(int64_t n_rows) { return tuning().fp4 && tuning().cta_group == 2 && n_rows < kFp4MaxN; }
int prefetch_dist() { return tuning().prefetch; }
int l2_hint() { return tuning().l2_hint; }
int tile_band() { return tuning().band > 0 ? tuning().band : 8; }

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
// become s units each so that r * s of the clusters share it instead of r.
// Short K (< kTailKMinKb k-blocks; latency-bound): column slices of the tile
// with the full K range, s a power of two, slices >= 32 wide.  Long K (the
// slices would be load-bound: a narrow MMA still streams a full A block):
// K ranges of the full tile, s = clusters / r, whose int32 partials are summed
// by e <= s epilogue units, one column slice each (config 3: 820 tiles = 11
// rounds of 74 + 6; the 6 run as 72 K ranges, summed by 48 epilogue slices).
// Knob "tail": 0 off, 1 auto, 2 slices only, 3 K ranges only.
constexpr int kTailKMinKb = 256;
struct TailPlan {
    int n_full, split, kmode, epi;
};
TailPlan tail_plan(int64_t n_tiles, int cg, int clusters, int nkb) {
    TailPlan tp{(int)n_tiles, 1, 0, 1};
    const int mode = tuning().tail;
    if (!mode || clusters < 2) return tp;
    const int64_t r = n_tiles % clusters;
    if (r == 0) return tp;
    const bool kmode = mode == 3 || (mode == 1 && nkb >= kTailKMinKb);
    int s = 1, e = 1;
    while (e * 2 * 32 <= 128 * cg && r * e * 2 <= clusters) e *= 2;  // power-of-two column slices
    if (kmode) {
        s = (int)(clusters / r);
        if (s > nkb) s = nkb;
        if (s > kTailMaxUnits) s = kTailMaxUnits;
        while (e > s) e /= 2;  // epilogue slices stay a power of two
    } else {
        s = e;
    }
    if (s < 2 || r * s > kTailMaxUnits) return tp;
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

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct DevInfo {
    int num_sms = 0;
    int major = 0;
    int minor = 0;
};

std::mutex g_info_mu;
DevInfo g_info[64];

int query_device(int device, DevInfo* out) {
    if (device < 0 || device >= 64) return fail(MI_ERR_UNSUPPORTED, "bad device ordinal %d", device);
    std::lock_guard<std::mutex> lk(g_info_mu);
    DevInfo& d = g_info[device];
    if (d.num_sms == 0) {
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess || n <= device)
            return fail(MI_ERR_UNSUPPORTED, "no CUDA device %d (%s)", device,
                        e == cudaSuccess ? "not present" : cudaGetErrorString(e));
        MI_CUDA(cudaDeviceGetAttribute(&d.num_sms, cudaDevAttrMultiProcessorCount, device));
        MI_CUDA(cudaDeviceGetAttribute(&d.major, cudaDevAttrComputeCapabilityMajor, device));
        MI_CUDA(cudaDeviceGetAttribute(&d.minor, cudaDevAttrComputeCapabilityMinor, device));
    }
    *out = d;
    if (d.major != 10 || d.minor != 0)
        return fail(MI_ERR_UNSUPPORTED, "device %d is sm_%d%d; this engine is built for sm_100a only",
                    device, d.major, d.minor);
    return MI_OK;
}

int current_device_info(DevInfo* out) {
    int dev = 0;
    MI_CUDA(cudaGetDevice(&dev));
    return query_device(dev, out);
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

// The fixed-point c log2 c table follows the per-column stats in the colstat
// workspace (see mi_colstat_bytes); nullptr when N is beyond the table path.
long long* xlogx_ptr(void* colstat, int64_t n_rows, int64_t n_cols) {
    if (n_rows < 1 || n_rows >= kXlogxMaxN) return nullptr;
    return reinterpret_cast<long long*>(reinterpret_cast<char*>(colstat) +
                                        mi_kmajor_rows(n_cols) * (int64_t)sizeof(ColStat));
}

// Per-128-column (min, max) column sums, after the table.
int2* blkrange_ptr(void* colstat, int64_t n_rows, int64_t n_cols) {
    long long* t = xlogx_ptr(colstat, n_rows, n_cols);
    return t ? reinterpret_cast<int2*>(t + n_rows + 1) : nullptr;
}

// fix_xlog2x's mantissa tables (kFixR, kFixLG) in global memory, after the
// block ranges: the hybrid epilogue evaluates T(c00) with them through L1.
float* fixr_ptr(void* colstat, int64_t n_rows, int64_t n_cols) {
    int2* b = blkrange_ptr(colstat, n_rows, n_cols);
    return b ? reinterpret_cast<float*>(b + mi_kmajor_rows(n_cols) / 128) : nullptr;
}

// rcp = round(2^(62 + nb) / N) and off0 = -(nb - 2) - s for fixed_to_fp
void fixed_point_consts(int64_t N, unsigned long long* rcp, int* off0) {
    int nb = 0;
    while (nb < 63 && (1ll << nb) <= N) ++nb;
    const unsigned __int128 num = (unsigned __int128)1 << (62 + nb);
    *rcp = (unsigned long long)((num + (unsigned __int128)(N / 2)) / (unsigned __int128)N);
    *off0 = -(nb - 2) - xlogx_scale(N);
}

int check_shape(int64_t n_rows, int64_t n_cols) {
    if (n_rows < 1 || n_cols < 1)
        return fail(MI_ERR_DIMENSION, "matrix must have at least one row and one column");
    if (n_rows > 0x7FFFFFFFLL) return fail(MI_ERR_DIMENSION, "n_rows %lld exceeds 2^31-1", (long long)n_rows);
    if (n_cols > 0x7FFFFFFFLL) return fail(MI_ERR_DIMENSION, "n_cols %lld exceeds 2^31-1", (long long)n_cols);
    return MI_OK;
}

int check_mode(int mode, double eps, int out_kind) {
    if (mode != MI_MODE_EXACT && mode != MI_MODE_EPSILON)
        return fail(MI_ERR_DOMAIN, "mode must be exact (0) or epsilon (1), got %d", mode);
    if (!(eps > 0.0)) return fail(MI_ERR_DOMAIN, "epsilon must be positive, got %g", eps);
    if (out_kind != MI_OUT_COUNTS && out_kind != MI_OUT_F64 && out_kind != MI_OUT_F32)
        return fail(MI_ERR_DOMAIN, "unknown output kind %d", out_kind);
    return MI_OK;
}

// binmat.py:78-80: padding bits beyond the last row must be zero
int check_padding(const uint64_t* h_words, int64_t n_rows, int64_t n_cols) {
    const int64_t nw = (n_rows + 63) / 64;
    const int rem = (int)(n_rows % 64);
    if (rem == 0) return MI_OK;
    const uint64_t pad = ~((1ull << rem) - 1ull);
    for (int64_t c = 0; c < n_cols; ++c)
        if (h_words[c * nw + nw - 1] & pad)
            return fail(MI_ERR_DOMAIN, "padding bits beyond the last row must be zero (column %lld)",
                        (long long)c);
    return MI_OK;
}

// Tile rows/columns that contain real columns (the operand is padded to 256).
int64_t tiles_per_side(int64_t n_cols) {
    const int64_t t = mi_tile_size();
    return (n_cols + t - 1) / t;
}

// Banded upper-triangle order: within a band of `band` tile rows, sweep J and
// then the band's rows, so tiles that run concurrently share operand blocks.
// `first` > 0 makes the first band that many rows (1 for the host path: tile
// row 0 completes in the first wave, so the D2H of finished rows starts early).
std::vector<int32_t> all_tiles(int64_t T, int band, int first = 0) {
    std::vector<int32_t> v;
    v.reserve((size_t)(T * (T + 1)));
    for (int64_t I0 = 0; I0 < T;) {
        const int64_t b = (I0 == 0 && first > 0) ? first : band;
        for (int64_t J = I0; J < T; ++J)
            for (int64_t I = I0; I < I0 + b && I <= J; ++I) {
                v.push_back((int32_t)I);
                v.push_back((int32_t)J);
            }
        I0 += b;
    }
    return v;
}

// A rank's tiles.  Round robin over the banded order (every rank touches
// nearly every column block), except for 8 ranks ("shard" knob, T >= 8): the
// column blocks form 4 groups; ranks 0-5 take the 6 off-diagonal group pairs
// (g, h), ranks 6 and 7 two diagonal groups each ((0,0)+(3,3), (1,1)+(2,2)).
// Every rank then reads -- and unpacks -- only 2 of the 4 groups (half of X),
// at a load imbalance of ~4/T (off-diagonal s^2 tiles vs s^2 + s).
std::vector<int32_t> rank_tiles(int64_t T, int rank, int world, int band) {
    const std::vector<int32_t> all = all_tiles(T, band);
    const int64_t total = (int64_t)all.size() / 2;
    std::vector<int32_t> v;
    if (world == 8 && T >= 8 && tuning().shard) {
        auto group = [&](int64_t b) { return (int)((b * 4) / T); };
        static const int pairs[8][4] = {{0, 1, -1, -1}, {0, 2, -1, -1}, {0, 3, -1, -1}, {1, 2, -1, -1},
                                        {1, 3, -1, -1}, {2, 3, -1, -1}, {0, 0, 3, 3}, {1, 1, 2, 2}};
        std::vector<std::vector<int32_t>> share(8);
        for (int64_t k = 0; k < total; ++k) {
            const int gi = group(all[2 * k]), gj = group(all[2 * k + 1]);
            for (int r = 0; r < 8; ++r) {
                const int* pr = pairs[r];
                if ((gi == pr[0] && gj == pr[1]) || (pr[2] >= 0 && gi == pr[2] && gj == pr[3])) {
                    share[r].push_back(all[2 * k]);
                    share[r].push_back(all[2 * k + 1]);
                    break;
                }
            }
        }
        // The two diagonal-group ranks hold s(s + 1) tiles against s^2: hand
        // their surplus (from the end of their lists) to off-diagonal ranks
        // that already hold that group's blocks -- no extra unpack -- always
        // to the least loaded one, until no rank exceeds ceil(total / 8).
        const size_t cap = (size_t)((total + 7) / 8);
        auto holds = [&](int r, int g) { return pairs[r][0] == g || pairs[r][1] == g; };
        for (int d = 6; d < 8; ++d) {
            while (share[d].size() / 2 > cap) {
                int best_r = -1;
                int64_t best_k = -1;
                for (int gsel = 0; gsel < 2; ++gsel) {
                    const int g = pairs[d][2 * gsel];
                    int r_min = -1;
                    for (int r = 0; r < 6; ++r)
                        if (holds(r, g) && (r_min < 0 || share[r].size() < share[r_min].size())) r_min = r;
                    if (r_min < 0 || share[r_min].size() / 2 >= cap) continue;
                    if (best_r >= 0 && share[best_r].size() <= share[r_min].size()) continue;
                    for (int64_t k = (int64_t)share[d].size() / 2 - 1; k >= 0; --k)
                        if (group(share[d][2 * k]) == g) {
                            best_r = r_min;
                            best_k = k;
                            break;
                        }
                }
                if (best_r < 0) break;
                share[best_r].push_back(share[d][2 * best_k]);
                share[best_r].push_back(share[d][2 * best_k + 1]);
                share[d].erase(share[d].begin() + 2 * best_k, share[d].begin() + 2 * best_k + 2);
            }
        }
        return share[rank];
    }
    for (int64_t g = rank; g < total; g += world) {
        v.push_back(all[2 * g]);
        v.push_back(all[2 * g + 1]);
    }
    return v;
}

// Grow-only device workspace for the host-buffer entry points.
struct Workspace {
    int device = -1;
    cudaStream_t stream = nullptr;
    void* words = nullptr; size_t words_cap = 0;
    void* x = nullptr; size_t x_cap = 0;
    void* colsum = nullptr; size_t colsum_cap = 0;
    void* colstat = nullptr; size_t colstat_cap = 0;
    void* tiles = nullptr; size_t tiles_cap = 0;
    void* out = nullptr; size_t out_cap = 0;
    void* h_stage = nullptr; size_t h_stage_cap = 0;  // pinned staging of pageable host words
    cudaStream_t copy_stream = nullptr;   // D2H of finished row bands
    cudaEvent_t copy_ev[2] = {nullptr, nullptr};  // the last two D2H copies
    cudaEvent_t stage_ev[kMaxIngestStages] = {};  // staged path: stage g's tiles are stored
    unsigned int* row_done_h = nullptr;   // pinned, mapped: per tile row completion counts
    unsigned int* row_done_d = nullptr;   // device alias of row_done_h
    size_t row_done_cap = 0;
};
std::mutex g_ws_mu;
Workspace g_ws[64];

int ensure(void** p, size_t* cap, size_t need) {
    if (*cap >= need && *p) return MI_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    MI_CUDA(cudaMalloc(p, need ? need : 16));
    *cap = need;
    return MI_OK;
}

void release(Workspace& w) {
    if (w.device < 0) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(w.device);
    void** ps[] = {&w.words, &w.x, &w.colsum, &w.colstat, &w.tiles, &w.out};
    for (void** p : ps)
        if (*p) cudaFree(*p), *p = nullptr;
    w.words_cap = w.x_cap = w.colsum_cap = w.colstat_cap = w.tiles_cap = w.out_cap = 0;
    if (w.stream) cudaStreamDestroy(w.stream), w.stream = nullptr;
    if (w.copy_stream) cudaStreamDestroy(w.copy_stream), w.copy_stream = nullptr;
    for (auto& e : w.copy_ev)
        if (e) cudaEventDestroy(e), e = nullptr;
    for (auto& e : w.stage_ev)
        if (e) cudaEventDestroy(e), e = nullptr;
    if (w.row_done_h) cudaFreeHost(w.row_done_h), w.row_done_h = nullptr, w.row_done_d = nullptr;
    if (w.h_stage) cudaFreeHost(w.h_stage), w.h_stage = nullptr;
    w.h_stage_cap = 0;
    w.row_done_cap = 0;
    w.device = -1;
    cudaSetDevice(prev);
}

// words (host) -> X, colsum on the device; shared by the host entry points.
// True when h points into page-locked (or registered / managed) host memory
// that the copy engines can read directly.
bool host_is_pinned(const void* h) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

// memcpy with up to `threads` host threads (pageable -> pinned staging): one
// thread reaches ~10 GB/s, well short of the link's ~55.  The workers are a
// small persistent pool (created on first use, never torn down: spawning 8
// threads per group cost ~1 ms a call); calls are serialised by g_ws_mu.
struct CopyPool {
    std::mutex mu;
    std::condition_variable cv, done_cv;
    std::vector<std::thread> workers;
    struct Job { char* dst; const char* src; size_t n; };
    std::vector<Job> jobs;
    size_t next = 0, pending = 0;
    void ensure(int n) {
        while ((int)workers.size() < n) {
            workers.emplace_back([this] {
                for (;;) {
                    Job j;
                    {
                        std::unique_lock<std::mutex> lk(mu);
                        cv.wait(lk, [this] { return next < jobs.size(); });
                        j = jobs[next++];
                    }
                    memcpy(j.dst, j.src, j.n);
                    std::lock_guard<std::mutex> lk(mu);
                    if (--pending == 0) done_cv.notify_all();
                }
            });
            workers.back().detach();
        }
    }
};
CopyPool& copy_pool() {
    static CopyPool* p = new CopyPool();  // leaked on purpose: detached workers outlive static destruction
    return *p;
}

void parallel_memcpy(void* dst, const void* src, size_t bytes, int threads) {
    const size_t min_chunk = (size_t)4 << 20;
    const int t = (int)std::min<size_t>((size_t)threads, (bytes + min_chunk - 1) / min_chunk);
    if (t <= 1) {
        memcpy(dst, src, bytes);
        return;
    }
    CopyPool& pool = copy_pool();
    pool.ensure(t);
    const size_t chunk = (bytes + t - 1) / t;
    {
        std::lock_guard<std::mutex> lk(pool.mu);
        pool.jobs.clear();
        pool.next = 0;
        for (int i = 0; i < t; ++i) {
            const size_t o = (size_t)i * chunk;
            if (o >= bytes) break;
            pool.jobs.push_back({(char*)dst + o, (const char*)src + o, std::min(chunk, bytes - o)});
        }
        pool.pending = pool.jobs.size();
    }
    pool.cv.notify_all();
    std::unique_lock<std::mutex> lk(pool.mu);
    pool.done_cv.wait(lk, [&] { return pool.pending == 0; });
}

// H2D of host words into ws.words on ws.stream.  Pageable words (numpy
// arrays) go through the cached pinned staging buffer in 4 column chunks:
// host threads copy chunk k while the copy engine moves chunk k - 1 (the
// driver's own pageable path runs at ~10 GB/s).
int upload_words(Workspace& ws, const uint64_t* h_words, int64_t n_cols, int64_t nw) {
    const size_t bytes = (size_t)(n_cols * nw * 8);
    if (host_is_pinned(h_words)) {
        MI_CUDA(cudaMemcpyAsync(ws.words, h_words, bytes, cudaMemcpyHostToDevice, ws.stream));
        return MI_OK;
    }
    if (ws.h_stage_cap < bytes) {
        if (ws.h_stage) cudaFreeHost(ws.h_stage);
        ws.h_stage = nullptr;
        ws.h_stage_cap = 0;
        MI_CUDA(cudaHostAlloc(&ws.h_stage, bytes, cudaHostAllocDefault));
        ws.h_stage_cap = bytes;
    }
    const int threads = std::max(1, std::min(16, env_int("MI_B200_COPY_THREADS", 8)));
    const int64_t chunks = n_cols >= 4 ? 4 : 1;
    for (int64_t k = 0; k < chunks; ++k) {
        const int64_t c0 = n_cols * k / chunks, c1 = n_cols * (k + 1) / chunks;
        const size_t off = (size_t)(c0 * nw * 8), len = (size_t)((c1 - c0) * nw * 8);
        parallel_memcpy((char*)ws.h_stage + off, (const char*)h_words + off, len, threads);
        MI_CUDA(cudaMemcpyAsync((char*)ws.words + off, (char*)ws.h_stage + off, len, cudaMemcpyHostToDevice,
                                ws.stream));
    }
    return MI_OK;
}

int stage_inputs(Workspace& ws, const uint64_t* h_words, int64_t n_rows, int64_t n_cols, int64_t* ld_out,
                 int64_t* m_pad_out, const DevInfo& info) {
    const int64_t nw = (n_rows + 63) / 64;
    const int64_t ld = mi_kmajor_ld(n_rows);
    const int64_t m_pad = mi_kmajor_rows(n_cols);
    int rc;
    if ((rc = ensure(&ws.words, &ws.words_cap, (size_t)(n_cols * nw * 8)))) return rc;
    if ((rc = ensure(&ws.x, &ws.x_cap, (size_t)(m_pad * ld)))) return rc;
    if ((rc = ensure(&ws.colsum, &ws.colsum_cap, (size_t)(m_pad * 4)))) return rc;
    if ((rc = ensure(&ws.colstat, &ws.colstat_cap, (size_t)mi_colstat_bytes(n_rows, n_cols)))) return rc;
    if ((rc = upload_words(ws, h_words, n_cols, nw))) return rc;
    MI_CUDA(launch_unpack_colsum((const uint64_t*)ws.words, n_rows, n_cols, nw, (int8_t*)ws.x, ld, m_pad,
                                 (int32_t*)ws.colsum, (ColStat*)ws.colstat, xlogx_ptr(ws.colstat, n_rows, n_cols),
                                 blkrange_ptr(ws.colstat, n_rows, n_cols), fixr_ptr(ws.colstat, n_rows, n_cols),
                                 operand_fp4(n_rows), nullptr,
                                 mi_tile_size(), info.num_sms, ws.stream));
    *ld_out = ld;
    *m_pad_out = m_pad;
    return MI_OK;
}

int workspace_for(int device, Workspace** out, DevInfo* info) {
    int rc = query_device(device, info);
    if (rc) return rc;
    MI_CUDA(cudaSetDevice(device));
    Workspace& ws = g_ws[device];
    if (ws.device < 0) {
        ws.device = device;
        MI_CUDA(cudaStreamCreateWithFlags(&ws.stream, cudaStreamNonBlocking));
        MI_CUDA(cudaStreamCreateWithFlags(&ws.copy_stream, cudaStreamNonBlocking));
    }
    *out = &ws;
    return MI_OK;
}

int run_fused(Workspace& ws, int64_t n_rows, int64_t n_cols, int64_t ld, int64_t m_pad, int mode, double eps,
              int include_diagonal, int out_kind, void* d_out, int64_t ld_out, const DevInfo& info,
              unsigned int* row_done = nullptr) {
    (void)m_pad;
    const int64_t n_tiles = mi_num_tiles(n_cols);
    std::vector<int32_t> tiles = all_tiles(tiles_per_side(n_cols), tile_band(), row_done ? 1 : 0);
    int rc;
    if ((rc = ensure(&ws.tiles, &ws.tiles_cap, tiles.size() * 4))) return rc;
    MI_CUDA(cudaMemcpyAsync(ws.tiles, tiles.data(), tiles.size() * 4, cudaMemcpyHostToDevice, ws.stream));
    (void)info;
    return launch_fused((const int8_t*)ws.x, ws.colstat, n_rows, n_cols, ld, mode, eps, include_diagonal, out_kind,
                        d_out, ld_out, (const int32_t*)ws.tiles, n_tiles, row_done, ws.stream);
}

}  // namespace

// =========================================================================== C ABI
extern "C" {

int mi_b200_abi_version(void) { return MI_B200_ABI_VERSION; }

const char* mi_last_error(void) { return g_err; }

int mi_device_info(int device, int* num_sms, int* cc_major, int* cc_minor) {
    DevInfo d;
    int rc = query_device(device, &d);
    if (num_sms) *num_sms = d.num_sms;
    if (cc_major) *cc_major = d.major;
    if (cc_minor) *cc_minor = d.minor;
    return rc;
}

int64_t mi_kmajor_ld(int64_t n_rows) {
    const int64_t n = n_rows < 1 ? 1 : n_rows;
    return operand_fp4(n) ? round_up(n, 256) / 2 : round_up(n, 128);
}

int64_t mi_kmajor_rows(int64_t n_cols) { return round_up(n_cols < 1 ? 1 : n_cols, 256); }

int64_t mi_colstat_bytes(int64_t n_rows, int64_t n_cols) {
    const int64_t stats = mi_kmajor_rows(n_cols) * (int64_t)sizeof(ColStat);
    const int64_t table = (n_rows >= 1 && n_rows < kXlogxMaxN)
                              ? (n_rows + 1) * 8 + mi_kmajor_rows(n_cols) / 128 * 8 + kFixTabBytes
                              : 0;
    return stats + table;
}

int mi_tile_size(void) { return gram_mi_tile_size(cta_group()); }

int64_t mi_num_tiles(int64_t n_cols) {
    const int64_t T = tiles_per_side(n_cols);
    return T * (T + 1) / 2;
}

int64_t mi_tile_list(int64_t n_cols, int rank, int world, int band, int32_t* tiles_out, int64_t capacity) {
    if (n_cols < 1) return -fail(MI_ERR_DIMENSION, "n_cols must be >= 1");
    if (world < 1 || rank < 0 || rank >= world)
        return -fail(MI_ERR_DOMAIN, "bad rank %d of world %d", rank, world);
    if (band <= 0) band = tile_band();
    const int64_t T = tiles_per_side(n_cols);
    const std::vector<int32_t> mine = rank_tiles(T, rank, world, band);
    const int64_t count = (int64_t)mine.size() / 2;
    if (tiles_out) {
        if (count > capacity) return -fail(MI_ERR_DIMENSION, "tile buffer too small");
        memcpy(tiles_out, mine.data(), mine.size() * sizeof(int32_t));
    }
    return count;
}

int64_t mi_rank_blocks(int64_t n_cols, int rank, int world, uint8_t* mask_out, int64_t capacity) {
    if (n_cols < 1) return -fail(MI_ERR_DIMENSION, "n_cols must be >= 1");
    if (world < 1 || rank < 0 || rank >= world)
        return -fail(MI_ERR_DOMAIN, "bad rank %d of world %d", rank, world);
    const int64_t T = tiles_per_side(n_cols);
    if (!mask_out) return T;
    if (capacity < T) return -fail(MI_ERR_DIMENSION, "mask buffer too small");
    memset(mask_out, 0, (size_t)T);
    const std::vector<int32_t> mine = rank_tiles(T, rank, world, tile_band());
    for (size_t k = 0; k < mine.size(); ++k) mask_out[mine[k]] = 1;
    int64_t used = 0;
    for (int64_t b = 0; b < T; ++b) used += mask_out[b];
    return used;
}

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
    if (c_begin < 0 || c_begin % 32 || c_end > m_pad || c_begin >= c_end)
        return fail(MI_ERR_DIMENSION, "column range [%lld, %lld) must start at a multiple of 32 and lie in [0, %lld)",
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

int launch_fused(const int8_t* d_kmajor, const void* d_colstat, int64_t n_rows, int64_t n_cols, int64_t ld, int mode,
                 double epsilon, int include_diagonal, int out_kind, void* d_out, int64_t ld_out, const int32_t* d_tiles,
                 int64_t n_tiles, unsigned int* row_done, cudaStream_t stream) {
    int rc = check_shape(n_rows, n_cols);
    if (rc) return rc;
    if ((rc = check_mode(mode, epsilon, out_kind))) return rc;
    if (ld < mi_kmajor_ld(n_rows) || ld % 128)
        return fail(MI_ERR_DIMENSION, "ld %lld must be a multiple of 128 and >= %lld", (long long)ld,
                    (long long)mi_kmajor_ld(n_rows));
    if (ld_out != MI_PACKED_UPPER && ld_out < n_cols)
        return fail(MI_ERR_DIMENSION, "ld_out %lld < n_cols (or MI_PACKED_UPPER)", (long long)ld_out);
    if (n_tiles < 0 || n_tiles > 0x7FFFFFFF) return fail(MI_ERR_DIMENSION, "bad n_tiles");
    if (n_tiles == 0) return MI_OK;
    if (out_kind == MI_OUT_COUNTS && mode != MI_MODE_EXACT)
        return fail(MI_ERR_DOMAIN, "counts export ignores the mode; pass MI_MODE_EXACT");
    if ((reinterpret_cast<uintptr_t>(d_kmajor) & 15) != 0)
        return fail(MI_ERR_DOMAIN, "kmajor operand must be 16-byte aligned");
    DevInfo info;
    if ((rc = current_device_info(&info))) return rc;
    CUtensorMap tm;
    if ((rc = make_tmap(&tm, d_kmajor, ld, mi_kmajor_rows(n_cols)))) return rc;
    GramMiParams p;
    p.colstat = reinterpret_cast<const ColStat*>(d_colstat);
    p.tiles = reinterpret_cast<const int2*>(d_tiles);
    p.n_tiles = (int)n_tiles;
    p.num_k_blocks = (int)(mi_kmajor_ld(n_rows) / 128);
    p.n_rows = (int)n_rows;
    p.m = (int)n_cols;
    p.ld_out = ld_out;
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
    p.pace_window = pace_window(n_tiles, p.num_k_blocks, info.num_sms);
    if (p.pace_window > 0 && (rc = pace_slots(dev, &p.pace))) return rc;
    const TailPlan tp = tail_plan(n_tiles, cta_group(), info.num_sms / cta_group(), p.num_k_blocks);
    p.n_full = tp.n_full;
    p.tail_split = tp.split;
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
    MI_CUDA(launch_gram_mi(cta_group(), operand_fp4(n_rows), out_kind, eff_mode, tuning().stages, tuning().epi_warps,
                           tm, p, info.num_sms, stream));
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

int all_pairs_host_impl(const uint64_t* h_words, int64_t n_rows, int64_t n_cols, int mode, double epsilon,
                        int include_diagonal, int out_kind, void* h_out, int device, bool packed);

int mi_all_pairs_host(const uint64_t* h_words, int64_t n_rows, int64_t n_cols, int mode, double epsilon,
                      int include_diagonal, int out_kind, void* h_out, int device) {
    return all_pairs_host_impl(h_words, n_rows, n_cols, mode, epsilon, include_diagonal, out_kind, h_out, device,
                               false);
}

int mi_all_pairs_host_packed(const uint64_t* h_words, int64_t n_rows, int64_t n_cols, int mode, double epsilon,
                             int include_diagonal, int out_kind, void* h_out, int device) {
    return all_pairs_host_impl(h_words, n_rows, n_cols, mode, epsilon, include_diagonal, out_kind, h_out, device,
                               true);
}

// Staged ingest -> compute -> egress (full-matrix output): the column blocks
// are cut into S groups; group g's words go H2D and are unpacked, then the
// tiles whose larger block falls in group g run (all their operands are
// resident), and the region they complete -- rows [0, c0) x columns [c0, c1)
// and rows [c0, c1) x columns [0, c1) -- goes D2H on the copy stream while
// group g + 1 uploads and computes.  The egress (PCIe D2H of m^2 elements,
// the floor of this call) then starts after 1/S of the upload instead of all
// of it.
int all_pairs_host_staged(Workspace& ws, const uint64_t* h_words, int64_t n_rows, int64_t n_cols, int mode,
                          double epsilon, int include_diagonal, int out_kind, void* h_out, const DevInfo& info,
                          int stages) {
    const int64_t nw = (n_rows + 63) / 64;
    const int64_t ld = mi_kmajor_ld(n_rows);
    const int64_t m_pad = mi_kmajor_rows(n_cols);
    const int tile = mi_tile_size();
    const int64_t T = tiles_per_side(n_cols);
    int S = (int)(stages < T ? stages : T);
    const size_t esz = out_kind == MI_OUT_F64 ? 8 : 4;
    // group boundaries in blocks: even (ingest_split 0), or doubling (1:
    // T/2^(S-1), ..., T/4, T/2, T).  Doubling starts the egress after a small
    // first upload and leaves half of the matrix to the last group, whose
    // rows go down as one linear copy; even groups make 3/4 of it 2-D copies.
    std::vector<int64_t> blk;
    blk.push_back(0);
    for (int g = 1; g <= S; ++g) {
        const int64_t b = tuning().ingest_split ? (T >> (S - g)) : T * g / S;
        if (b > blk.back()) blk.push_back(b);
    }
    if (blk.back() != T) blk.push_back(T);
    S = (int)blk.size() - 1;
    int rc;
    if ((rc = ensure(&ws.words, &ws.words_cap, (size_t)(n_cols * nw * 8)))) return rc;
    if ((rc = ensure(&ws.x, &ws.x_cap, (size_t)(m_pad * ld)))) return rc;
    if ((rc = ensure(&ws.colsum, &ws.colsum_cap, (size_t)(m_pad * 4)))) return rc;
    if ((rc = ensure(&ws.colstat, &ws.colstat_cap, (size_t)mi_colstat_bytes(n_rows, n_cols)))) return rc;
    if ((rc = ensure(&ws.out, &ws.out_cap, (size_t)n_cols * (size_t)n_cols * esz))) return rc;
    // per-stage tile lists (banded order restricted to J in the group), one upload
    const std::vector<int32_t> all = all_tiles(T, tile_band(), 0);
    std::vector<int32_t> lists;
    std::vector<int64_t> first(S + 1, 0);
    for (int g = 0; g < S; ++g) {
        first[g] = (int64_t)lists.size() / 2;
        for (size_t k = 0; k < all.size(); k += 2)
            if (all[k + 1] >= blk[g] && all[k + 1] < blk[g + 1]) {
                lists.push_back(all[k]);
                lists.push_back(all[k + 1]);
            }
    }
    first[S] = (int64_t)lists.size() / 2;
    if ((rc = ensure(&ws.tiles, &ws.tiles_cap, lists.size() * 4))) return rc;
    MI_CUDA(cudaMemcpyAsync(ws.tiles, lists.data(), lists.size() * 4, cudaMemcpyHostToDevice, ws.stream));
    for (int g = 0; g < S; ++g)
        if (!ws.stage_ev[g]) MI_CUDA(cudaEventCreateWithFlags(&ws.stage_ev[g], cudaEventDisableTiming));
    ColStat* cs = (ColStat*)ws.colstat;
    long long* xl = xlogx_ptr(ws.colstat, n_rows, n_cols);
    int2* br = blkrange_ptr(ws.colstat, n_rows, n_cols);
    const bool fp4 = operand_fp4(n_rows);
    MI_CUDA(launch_unpack_prep(n_rows, m_pad, cs, xl, br, fixr_ptr(ws.colstat, n_rows, n_cols), info.num_sms,
                               ws.stream));
    const size_t pitch = (size_t)n_cols * esz;
    // Pageable words (the drop-in's numpy arrays) copy at ~10 GB/s through the
    // driver's bounce buffer, one stage after another, which starved the
    // pipeline (config 3: 14 ms of upload).  Stage them into a pinned buffer
    // with host threads instead, group by group, so each group's H2D runs at
    // link speed while the next group is being copied.
    const uint64_t* src_words = h_words;
    const bool stage_host = !host_is_pinned(h_words);
    if (stage_host) {
        const size_t need = (size_t)(n_cols * nw * 8);
        if (ws.h_stage_cap < need) {
            if (ws.h_stage) cudaFreeHost(ws.h_stage);
            ws.h_stage = nullptr;
            ws.h_stage_cap = 0;
            MI_CUDA(cudaHostAlloc(&ws.h_stage, need, cudaHostAllocDefault));
            ws.h_stage_cap = need;
        }
        src_words = (const uint64_t*)ws.h_stage;
    }
    const int copy_threads = std::max(1, std::min(16, env_int("MI_B200_COPY_THREADS", 8)));
    // MI_B200_TIMELINE=1: per-stage event timeline on stderr (experiments only)
    const bool tl_on = env_int("MI_B200_TIMELINE", 0) != 0;
    std::vector<cudaEvent_t> tl;
    auto mark = [&](cudaStream_t st) {
        if (!tl_on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        tl.push_back(e);
    };
    mark(ws.stream);
    for (int g = 0; g < S; ++g) {
        const int64_t c0 = std::min<int64_t>(blk[g] * tile, n_cols), c1 = std::min<int64_t>(blk[g + 1] * tile, n_cols);
        if (stage_host)  // (the previous groups' H2D copies read other parts of the staging buffer)
            parallel_memcpy((uint64_t*)ws.h_stage + c0 * nw, h_words + c0 * nw, (size_t)((c1 - c0) * nw * 8),
                            copy_threads);
        MI_CUDA(cudaMemcpyAsync((uint64_t*)ws.words + c0 * nw, src_words + c0 * nw, (size_t)((c1 - c0) * nw * 8),
                                cudaMemcpyHostToDevice, ws.stream));
        mark(ws.stream);  // H2D g done
        const int64_t u1 = g == S - 1 ? m_pad : blk[g + 1] * tile;
        MI_CUDA(launch_unpack_range((const uint64_t*)ws.words, n_rows, n_cols, nw, (int8_t*)ws.x, ld, m_pad,
                                    (int32_t*)ws.colsum, cs, xl ? br : nullptr, fp4, nullptr, tile, blk[g] * tile, u1,
                                    info.num_sms, ws.stream));
        if ((rc = launch_fused((const int8_t*)ws.x, ws.colstat, n_rows, n_cols, ld, mode, epsilon, include_diagonal,
                               out_kind, ws.out, n_cols, (const int32_t*)ws.tiles + 2 * first[g],
                               first[g + 1] - first[g], nullptr, ws.stream)))
            return rc;
        MI_CUDA(cudaEventRecord(ws.stage_ev[g], ws.stream));
        mark(ws.stream);  // compute g done
        MI_CUDA(cudaStreamWaitEvent(ws.copy_stream, ws.stage_ev[g], 0));
        mark(ws.copy_stream);  // D2H g may start
        char* ho = (char*)h_out;
        const char* dv = (const char*)ws.out;
        if (c0 > 0 && c1 > c0)  // rows above the group, the group's columns
            MI_CUDA(cudaMemcpy2DAsync(ho + c0 * esz, pitch, dv + c0 * esz, pitch, (size_t)(c1 - c0) * esz,
                                      (size_t)c0, cudaMemcpyDeviceToHost, ws.copy_stream));
        // the group's rows, columns [0, c1); one linear copy when they are whole
        // rows (the last group): 2-D copies run at ~52 GB/s against ~57 GB/s
        // linear on this link (tools/d2h_2d.py)
        if (c1 > c0 && c1 == n_cols)
            MI_CUDA(cudaMemcpyAsync(ho + c0 * pitch, dv + c0 * pitch, (size_t)(c1 - c0) * pitch,
                                    cudaMemcpyDeviceToHost, ws.copy_stream));
        else if (c1 > c0)
            MI_CUDA(cudaMemcpy2DAsync(ho + c0 * pitch, pitch, dv + c0 * pitch, pitch, (size_t)c1 * esz,
                                      (size_t)(c1 - c0), cudaMemcpyDeviceToHost, ws.copy_stream));
        mark(ws.copy_stream);  // D2H g done
    }
    MI_CUDA(cudaStreamSynchronize(ws.copy_stream));
    MI_CUDA(cudaStreamSynchronize(ws.stream));
    if (tl_on) {
        for (size_t k = 1; k < tl.size(); ++k) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, tl[0], tl[k]);
            static const char* what[4] = {"H2D done", "compute done", "D2H start", "D2H done"};
            fprintf(stderr, "[timeline] stage %zu %-12s %8.3f ms\n", (k - 1) / 4, what[(k - 1) % 4], ms);
        }
        for (cudaEvent_t e : tl) cudaEventDestroy(e);
    }
    return MI_OK;
}

int all_pairs_host_impl(const uint64_t* h_words, int64_t n_rows, int64_t n_cols, int mode, double epsilon,
                        int include_diagonal, int out_kind, void* h_out, int device, bool packed) {
    int rc = check_shape(n_rows, n_cols);
    if (rc) return rc;
    if ((rc = check_mode(mode, epsilon, out_kind))) return rc;
    if (out_kind == MI_OUT_COUNTS) return fail(MI_ERR_DOMAIN, "use mi_gram_ones_host for counts");
    if ((rc = check_padding(h_words, n_rows, n_cols))) return rc;
    std::lock_guard<std::mutex> lk(g_ws_mu);
    const bool verbose = env_int("MI_B200_VERBOSE", 0) != 0;
    const auto t0 = std::chrono::steady_clock::now();
    auto stamp = [&](const char* what) {
        if (verbose)
            fprintf(stderr, "[mi_all_pairs_host] %8.3f ms %s\n",
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(), what);
    };
    Workspace* ws;
    DevInfo info;
    if ((rc = workspace_for(device, &ws, &info))) return rc;
    if (!packed && tuning().ingest > 0 && tiles_per_side(n_cols) > 1) {
        rc = all_pairs_host_staged(*ws, h_words, n_rows, n_cols, mode, epsilon, include_diagonal, out_kind, h_out,
                                   info, tuning().ingest);
        stamp("done (staged)");
        return rc;
    }
    int64_t ld, m_pad;
    if ((rc = stage_inputs(*ws, h_words, n_rows, n_cols, &ld, &m_pad, info))) return rc;
    stamp("H2D + unpack enqueued");
    const size_t esz = out_kind == MI_OUT_F64 ? 8 : 4;
    const size_t row_bytes = (size_t)n_cols * esz;
    // byte offset of row r's first element in the output (full or packed upper triangle)
    auto row_off = [&](int64_t r) -> size_t {
        return packed ? (size_t)(r * n_cols - (r * (r - 1)) / 2) * esz : (size_t)r * row_bytes;
    };
    if ((rc = ensure(&ws->out, &ws->out_cap, row_off(n_cols)))) return rc;
    // per-tile-row completion counters in pinned, mapped host memory
    const int tile = mi_tile_size();
    const int64_t T = tiles_per_side(n_cols);
    if (ws->row_done_cap < (size_t)T) {
        if (ws->row_done_h) cudaFreeHost(ws->row_done_h);
        ws->row_done_h = nullptr;
        ws->row_done_cap = 0;
        MI_CUDA(cudaHostAlloc((void**)&ws->row_done_h, (size_t)T * 4, cudaHostAllocMapped));
        MI_CUDA(cudaHostGetDevicePointer((void**)&ws->row_done_d, ws->row_done_h, 0));
        ws->row_done_cap = (size_t)T;
        stamp("row counters allocated");
    }
    volatile unsigned int* done = ws->row_done_h;
    for (int64_t I = 0; I < T; ++I) done[I] = 0;
    // completion count of tile row I: +1 per CTA per tile (I, J), or per
    // column slice of a split tail tile -- the same tile list and tail plan
    // that run_fused launches
    const unsigned cg = (unsigned)cta_group();
    std::vector<unsigned> expect((size_t)T, 0u);
    {
        const std::vector<int32_t> tl = all_tiles(T, tile_band(), 1);
        const int64_t nt = (int64_t)tl.size() / 2;
        const TailPlan tp = tail_plan(nt, (int)cg, info.num_sms / (int)cg, (int)(mi_kmajor_ld(n_rows) / 128));
        for (int64_t k = 0; k < nt; ++k) expect[(size_t)tl[2 * k]] += cg * (k >= tp.n_full ? (unsigned)tp.epi : 1u);
    }
    if ((rc = run_fused(*ws, n_rows, n_cols, ld, m_pad, mode, epsilon, include_diagonal, out_kind, ws->out,
                        packed ? MI_PACKED_UPPER : n_cols, info, ws->row_done_d)))
        return rc;
    stamp("fused kernel enqueued");
    // Stream finished rows to the host while the GEMM continues: rows of tile
    // row b are final once every tile row I <= b is complete (its own tiles
    // and all mirrors landing in it), so copy the completed prefix.
    // At most two copies in flight: while the link is busy the finished rows
    // accumulate, so chunks grow (a handful of copies in all; each extra copy
    // costs ~25 us of engine time, tools/d2h_streams.py), yet the queued one
    // keeps the copy engine from idling between them.
    const int64_t min_chunk_rows = (int64_t)((16u << 20) / row_bytes) + 1;  // (packed: rows shrink; fine)
    int64_t copied = 0, I = 0;
    bool kernel_done = false;
    if (!ws->copy_ev[0]) {
        MI_CUDA(cudaEventCreateWithFlags(&ws->copy_ev[0], cudaEventDisableTiming));
        MI_CUDA(cudaEventCreateWithFlags(&ws->copy_ev[1], cudaEventDisableTiming));
    }
    int issued = 0;
    auto in_flight = [&]() {
        int n = 0;
        for (int k = issued - 2 < 0 ? 0 : issued - 2; k < issued; ++k)
            if (cudaEventQuery(ws->copy_ev[k & 1]) == cudaErrorNotReady) ++n;
        return n;
    };
    while (copied < n_cols) {
        while (I < T && done[I] >= expect[(size_t)I]) ++I;
        int64_t final_rows = I * tile < n_cols ? I * tile : n_cols;
        if (kernel_done) final_rows = n_cols;
        if (final_rows > copied && (final_rows - copied >= min_chunk_rows || final_rows == n_cols) &&
            (kernel_done || in_flight() < 2)) {
            MI_CUDA(cudaMemcpyAsync((char*)h_out + row_off(copied), (char*)ws->out + row_off(copied),
                                    row_off(final_rows) - row_off(copied), cudaMemcpyDeviceToHost, ws->copy_stream));
            MI_CUDA(cudaEventRecord(ws->copy_ev[issued & 1], ws->copy_stream));
            ++issued;
            if (verbose) {
                char msg[96];
                snprintf(msg, sizeof(msg), "D2H rows [%lld, %lld) issued", (long long)copied, (long long)final_rows);
                stamp(msg);
            }
            copied = final_rows;
            continue;
        }
        const cudaError_t q = cudaStreamQuery(ws->stream);
        if (q == cudaSuccess) {
            kernel_done = true;  // everything is final now
        } else if (q != cudaErrorNotReady) {
            cudaStreamSynchronize(ws->copy_stream);
            return cuda_fail(q, "fused kernel");
        } else {
            std::this_thread::sleep_for(std::chrono::microseconds(20));
        }
    }
    MI_CUDA(cudaStreamSynchronize(ws->copy_stream));
    MI_CUDA(cudaStreamSynchronize(ws->stream));
    stamp("done");
    return MI_OK;
}

int mi_gram_ones_host(const uint64_t* h_words, int64_t n_cols, int64_t n_words, int64_t* h_out, int device) {
    if (n_cols < 1 || n_words < 1) return fail(MI_ERR_DIMENSION, "words must be a non-empty (m, nw) array");
    const int64_t n_rows = n_words * 64;  // padding bits are zero, so they add nothing
    std::lock_guard<std::mutex> lk(g_ws_mu);
    Workspace* ws;
    DevInfo info;
    int rc;
    if ((rc = workspace_for(device, &ws, &info))) return rc;
    int64_t ld, m_pad;
    if ((rc = stage_inputs(*ws, h_words, n_rows, n_cols, &ld, &m_pad, info))) return rc;
    const size_t out_bytes = (size_t)n_cols * (size_t)n_cols * 4;
    if ((rc = ensure(&ws->out, &ws->out_cap, out_bytes))) return rc;
    if ((rc = run_fused(*ws, n_rows, n_cols, ld, m_pad, MI_MODE_EXACT, 1e-12, 1, MI_OUT_COUNTS, ws->out, n_cols,
                        info)))
        return rc;
    std::vector<int32_t> tmp((size_t)n_cols * (size_t)n_cols);
    MI_CUDA(cudaMemcpyAsync(tmp.data(), ws->out, out_bytes, cudaMemcpyDeviceToHost, ws->stream));
    MI_CUDA(cudaStreamSynchronize(ws->stream));
    for (size_t k = 0; k < tmp.size(); ++k) h_out[k] = tmp[k];
    return MI_OK;
}

int mi_column_sums_host(const uint64_t* h_words, int64_t n_cols, int64_t n_words, uint64_t* h_out, int device) {
    if (n_cols < 1 || n_words < 1) return fail(MI_ERR_DIMENSION, "words must be a non-empty (m, nw) array");
    std::lock_guard<std::mutex> lk(g_ws_mu);
    Workspace* ws;
    DevInfo info;
    int rc;
    if ((rc = workspace_for(device, &ws, &info))) return rc;
    int64_t ld, m_pad;
    if ((rc = stage_inputs(*ws, h_words, n_words * 64, n_cols, &ld, &m_pad, info))) return rc;
    std::vector<int32_t> tmp((size_t)n_cols);
    MI_CUDA(cudaMemcpyAsync(tmp.data(), ws->colsum, (size_t)n_cols * 4, cudaMemcpyDeviceToHost, ws->stream));
    MI_CUDA(cudaStreamSynchronize(ws->stream));
    for (int64_t k = 0; k < n_cols; ++k) h_out[k] = (uint64_t)tmp[k];
    return MI_OK;
}

// ---------------------------------------------------------------- sharded egress

int mi_host_register(void* h_ptr, int64_t bytes) {
    if (!h_ptr || bytes < 1) return fail(MI_ERR_DOMAIN, "bad host range");
    MI_CUDA(cudaHostRegister(h_ptr, (size_t)bytes, cudaHostRegisterPortable));
    return MI_OK;
}

int mi_host_unregister(void* h_ptr) {
    if (!h_ptr) return fail(MI_ERR_DOMAIN, "null host pointer");
    MI_CUDA(cudaHostUnregister(h_ptr));
    return MI_OK;
}

// Tiles and their mirrors, device -> host, as few 2-D copies as possible: runs
// of consecutive J in a tile row merge, then identical runs in consecutive tile
// rows (an 8-rank column-group share is one or two rectangles).
int mi_copy_tiles_to_host(const void* d_out, int64_t ld_out, int64_t n_cols, int esz, const int32_t* h_tiles,
                          int64_t n_tiles, void* h_dst, int64_t ld_dst, void* stream) {
    if (!d_out || !h_dst || (n_tiles > 0 && !h_tiles)) return fail(MI_ERR_DOMAIN, "null argument");
    if (esz != 4 && esz != 8) return fail(MI_ERR_DOMAIN, "esz must be 4 or 8");
    if (ld_out < n_cols || ld_dst < n_cols) return fail(MI_ERR_DIMENSION, "pitch < n_cols");
    const int64_t t = mi_tile_size();
    const int64_t T = tiles_per_side(n_cols);
    std::vector<std::pair<int32_t, int32_t>> v;
    v.reserve((size_t)n_tiles);
    for (int64_t k = 0; k < n_tiles; ++k) {
        const int32_t I = h_tiles[2 * k], J = h_tiles[2 * k + 1];
        if (I < 0 || J < 0 || I >= T || J >= T) return fail(MI_ERR_DIMENSION, "tile (%d, %d) outside %lld", I, J, (long long)T);
        v.push_back({I, J});
    }
    std::sort(v.begin(), v.end());
    struct Run { int32_t I, J0, J1; };  // tile row I, tile columns [J0, J1)
    std::vector<Run> runs;
    for (size_t k = 0; k < v.size();) {
        size_t e = k + 1;
        while (e < v.size() && v[e].first == v[k].first && v[e].second == v[e - 1].second + 1) ++e;
        runs.push_back({v[k].first, v[k].second, v[e - 1].second + 1});
        k = e;
    }
    struct Rect { int32_t I0, I1, J0, J1; };
    std::vector<Rect> rects;
    for (const Run& r : runs) {
        if (!rects.empty() && rects.back().I1 == r.I && rects.back().J0 == r.J0 && rects.back().J1 == r.J1)
            rects.back().I1 = r.I + 1;
        else
            rects.push_back({r.I, r.I + 1, r.J0, r.J1});
    }
    cudaStream_t st = (cudaStream_t)stream;
    auto copy = [&](int64_t r0, int64_t r1, int64_t c0, int64_t c1) -> int {
        r1 = r1 < n_cols ? r1 : n_cols;
        c1 = c1 < n_cols ? c1 : n_cols;
        if (r0 >= r1 || c0 >= c1) return MI_OK;
        MI_CUDA(cudaMemcpy2DAsync((char*)h_dst + (r0 * ld_dst + c0) * esz, (size_t)(ld_dst * esz),
                                  (const char*)d_out + (r0 * ld_out + c0) * esz, (size_t)(ld_out * esz),
                                  (size_t)((c1 - c0) * esz), (size_t)(r1 - r0), cudaMemcpyDeviceToHost, st));
        return MI_OK;
    };
    int rc;
    for (const Rect& q : rects) {
        if ((rc = copy(q.I0 * t, q.I1 * t, q.J0 * t, q.J1 * t))) return rc;  // tiles
        if ((rc = copy(q.J0 * t, q.J1 * t, q.I0 * t, q.I1 * t))) return rc;  // mirrors
    }
    return MI_OK;
}

// ---------------------------------------------------------------- BMI1 ingest

int mi_bmi_header(const char* path, int64_t* n_rows, int64_t* n_cols) {
    if (!path || !n_rows || !n_cols) return fail(MI_ERR_DOMAIN, "null argument");
    FILE* f = fopen(path, "rb");
    if (!f) return fail(MI_ERR_FORMAT, "%s: cannot open", path);
    unsigned char h[20];
    const size_t got = fread(h, 1, 20, f);
    fseek(f, 0, SEEK_END);
    const long long size = ftell(f);
    fclose(f);
    if (got < 20) return fail(MI_ERR_FORMAT, "%s: file shorter than the 20-byte header", path);
    if (memcmp(h, "BMI1", 4) != 0) return fail(MI_ERR_FORMAT, "%s: bad magic, expected 'BMI1'", path);
    uint64_t nr = 0, nc = 0;
    for (int k = 7; k >= 0; --k) {
        nr = (nr << 8) | h[4 + k];
        nc = (nc << 8) | h[12 + k];
    }
    if (nr < 1 || nc < 1 || nr > (1ull << 40) || nc > (1ull << 31))
        return fail(MI_ERR_FORMAT, "%s: invalid dimensions %llux%llu", path, (unsigned long long)nr,
                    (unsigned long long)nc);
    const long long nw = (long long)((nr + 63) / 64);
    const long long expected = 20 + (long long)nc * nw * 8;
    if (size != expected)
        return fail(MI_ERR_FORMAT, "%s: payload length %lld does not match %llu columns of %lld words (%lld bytes)",
                    path, size - 20, (unsigned long long)nc, nw, expected - 20);
    *n_rows = (int64_t)nr;
    *n_cols = (int64_t)nc;
    return MI_OK;
}

int mi_bmi_load(const char* path, uint64_t* d_words, int64_t n_rows, int64_t n_cols, void* stream) {
    int64_t hr = 0, hc = 0;
    int rc = mi_bmi_header(path, &hr, &hc);
    if (rc) return rc;
    if (hr != n_rows || hc != n_cols)
        return fail(MI_ERR_DIMENSION, "%s holds %lldx%lld, caller expects %lldx%lld", path, (long long)hr,
                    (long long)hc, (long long)n_rows, (long long)n_cols);
    if (!d_words) return fail(MI_ERR_DOMAIN, "null device buffer");
    const int64_t nw = (n_rows + 63) / 64;
    const uint64_t pad = (n_rows % 64) ? ~((1ull << (n_rows % 64)) - 1) : 0ull;  // bits past the last row
    const int64_t total = n_cols * nw;                                              // words
    const int64_t chunk = (int64_t)8 << 20;                                         // words (64 MB)
    static std::mutex mu;
    static uint64_t* stage[2] = {nullptr, nullptr};
    static cudaEvent_t done[2];
    std::lock_guard<std::mutex> lk(mu);
    if (!stage[0]) {
        for (int b = 0; b < 2; ++b) {
            MI_CUDA(cudaHostAlloc((void**)&stage[b], (size_t)chunk * 8, cudaHostAllocDefault));
            MI_CUDA(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
            MI_CUDA(cudaEventRecord(done[b], 0));
        }
    }
    FILE* f = fopen(path, "rb");
    if (!f) return fail(MI_ERR_FORMAT, "%s: cannot open", path);
    fseek(f, 20, SEEK_SET);
    cudaStream_t st = (cudaStream_t)stream;
    int b = 0;
    for (int64_t w0 = 0; w0 < total; w0 += chunk, b ^= 1) {
        const int64_t n = total - w0 < chunk ? total - w0 : chunk;
        cudaError_t e = cudaEventSynchronize(done[b]);  // the copy that last used this buffer
        if (e != cudaSuccess) { fclose(f); return cuda_fail(e, "staging reuse"); }
        if ((int64_t)fread(stage[b], 8, (size_t)n, f) != n) {
            fclose(f);
            return fail(MI_ERR_FORMAT, "%s: short read", path);
        }
        if (pad) {  // the last word of every column in this chunk (little-endian host)
            int64_t first = w0 + (nw - 1 - w0 % nw + nw) % nw;
            for (int64_t w = first; w < w0 + n; w += nw)
                if (stage[b][w - w0] & pad) {
                    fclose(f);
                    return fail(MI_ERR_FORMAT, "%s: nonzero padding bits past row %lld", path, (long long)(n_rows - 1));
                }
        }
        e = cudaMemcpyAsync(d_words + w0, stage[b], (size_t)n * 8, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaEventRecord(done[b], st);
        if (e != cudaSuccess) { fclose(f); return cuda_fail(e, "BMI1 payload H2D"); }
    }
    fclose(f);
    MI_CUDA(cudaStreamSynchronize(st));
    return MI_OK;
}

int mi_set_tuning(const char* key, int value) {
    if (!key) return fail(MI_ERR_DOMAIN, "null tuning key");
    Tuning& t = tuning();
    if (!strcmp(key, "cta_group")) {
        if (value != 1 && value != 2) return fail(MI_ERR_DOMAIN, "cta_group must be 1 or 2");
        t.cta_group = value;
    } else if (!strcmp(key, "prefetch")) {
        if (value < 0 || value > 256) return fail(MI_ERR_DOMAIN, "prefetch must be in [0, 256]");
        t.prefetch = value;
    } else if (!strcmp(key, "l2_hint")) {
        if (value < 0 || value > 2) return fail(MI_ERR_DOMAIN, "l2_hint must be 0, 1 or 2");
        t.l2_hint = value;
    } else if (!strcmp(key, "band")) {
        if (value < 1) return fail(MI_ERR_DOMAIN, "band must be >= 1");
        t.band = value;
    } else if (!strcmp(key, "stages")) {
        if (value != 6) return fail(MI_ERR_DOMAIN, "stages must be 6");
        t.stages = value;
    } else if (!strcmp(key, "table_thr")) {
        t.table_thr = value;
    } else if (!strcmp(key, "fixed")) {
        if (value < 0 || value > 3) return fail(MI_ERR_DOMAIN, "fixed must be 0, 1, 2 or 3");
        t.fixed = value;
    } else if (!strcmp(key, "tail")) {
        if (value < 0 || value > 3) return fail(MI_ERR_DOMAIN, "tail must be 0 (off), 1 (auto), 2 (slices) or 3 (K ranges)");
        t.tail = value;
    } else if (!strcmp(key, "hybrid")) {
        if (value != 0 && value != 1) return fail(MI_ERR_DOMAIN, "hybrid must be 0 or 1");
        t.hybrid = value;
    } else if (!strcmp(key, "shard")) {
        if (value != 0 && value != 1) return fail(MI_ERR_DOMAIN, "shard must be 0 (round robin) or 1 (column groups)");
        t.shard = value;
    } else if (!strcmp(key, "evac")) {
        if (value < 0 || value > 2) return fail(MI_ERR_DOMAIN, "evac must be 0, 1 or 2");
        t.evac = value;
    } else if (!strcmp(key, "fp4")) {
        if (value != 0 && value != 1) return fail(MI_ERR_DOMAIN, "fp4 must be 0 (int8 operands) or 1");
        t.fp4 = value;
    } else if (!strcmp(key, "pace")) {
        if (value < -1) return fail(MI_ERR_DOMAIN, "pace must be -1 (auto), 0 (off) or a window in k-blocks");
        t.pace = value;
    } else if (!strcmp(key, "ingest")) {
        if (value < 0 || value > kMaxIngestStages)
            return fail(MI_ERR_DOMAIN, "ingest must be 0 (row-band egress) or 1..%d stages", kMaxIngestStages);
        t.ingest = value;
    } else if (!strcmp(key, "serp")) {
        if (value != 0 && value != 1) return fail(MI_ERR_DOMAIN, "serp must be 0 or 1");
        t.serp = value;
    } else if (!strcmp(key, "ingest_split")) {
        if (value != 0 && value != 1) return fail(MI_ERR_DOMAIN, "ingest_split must be 0 (even) or 1 (doubling)");
        t.ingest_split = value;
    } else if (!strcmp(key, "unperm_ctas")) {
        if (value < 0 || value > 4) return fail(MI_ERR_DOMAIN, "unperm_ctas must be 0 (auto) or 1..4");
        t.unperm_ctas = value;
    } else if (!strcmp(key, "f32_epi")) {
        if (value != 0 && value != 1) return fail(MI_ERR_DOMAIN, "f32_epi must be 0 (FP64) or 1 (FP32 pipe)");
        t.f32_epi = value;
    } else if (!strcmp(key, "epi_warps")) {
        if (value != 8 && value != 16) return fail(MI_ERR_DOMAIN, "epi_warps must be 8 or 16");
        t.epi_warps = value;
    } else {
        return fail(MI_ERR_DOMAIN, "unknown tuning key '%s'", key);
    }
    return MI_OK;
}

int mi_get_tuning(const char* key) {
    const Tuning& t = tuning();
    if (!key) return -1;
    if (!strcmp(key, "cta_group")) return t.cta_group;
    if (!strcmp(key, "prefetch")) return t.prefetch;
    if (!strcmp(key, "l2_hint")) return t.l2_hint;
    if (!strcmp(key, "band")) return t.band;
    if (!strcmp(key, "stages")) return t.stages;
    if (!strcmp(key, "epi_warps")) return t.epi_warps;
    if (!strcmp(key, "fixed")) return t.fixed;
    if (!strcmp(key, "table_thr")) return t.table_thr;
    if (!strcmp(key, "pace")) return t.pace;
    if (!strcmp(key, "tail")) return t.tail;
    if (!strcmp(key, "fp4")) return t.fp4;
    if (!strcmp(key, "evac")) return t.evac;
    if (!strcmp(key, "shard")) return t.shard;
    if (!strcmp(key, "hybrid")) return t.hybrid;
    if (!strcmp(key, "unperm_ctas")) return t.unperm_ctas;
    if (!strcmp(key, "ingest")) return t.ingest;
    if (!strcmp(key, "ingest_split")) return t.ingest_split;
    if (!strcmp(key, "serp")) return t.serp;
    if (!strcmp(key, "f32_epi")) return t.f32_epi;
    return -1;
}

// Not part of the public header: route per-tile timestamps of cluster 0 into a
// device buffer of 64 x 4 int64 (tools/trace_tiles.py) followed by 256 x 4
// per-cluster globaltimer stamps (start, main tiles done, tail done), or
// nullptr to stop.
void mi_debug_set_trace(void* d_buf) { g_trace = reinterpret_cast<long long*>(d_buf); }

void mi_release_workspace(void) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    for (auto& w : g_ws) release(w);
}

}  // extern "C"
