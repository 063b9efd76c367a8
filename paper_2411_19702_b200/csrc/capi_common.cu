// C-ABI layer, shared pieces: error state, tuning knobs, device queries,
// argument checks and the operand / workspace layout (declared in
// capi_internal.h; the public entry points are in include/mimatrix_b200.h).
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
#include "capi_internal.h"
#include "mi_kernels.h"
#include "milog.cuh"

using namespace mib200;
using namespace mib200::capi;

namespace mib200 {
namespace capi {


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


// Tuning knobs: defaults are the measured best; MI_B200_* env vars
// or mi_set_tuning() override them.  cta_group 2 = 256 x 256 tiles on a CTA
// pair (production); 1 = single-SM 128 x 128 tiles.

int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return (e && *e) ? atoi(e) : dflt;
}
Tuning& tuning() {
    static Tuning t = {env_int("MI_B200_CTA_GROUP", 2) == 1 ? 1 : 2, env_int("MI_B200_PREFETCH", 0),
                       env_int("MI_B200_L2HINT", 1), env_int("MI_B200_BAND", 8),
                       env_int("MI_B200_STAGES", 6), env_int("MI_B200_EPI_WARPS", 8), env_int("MI_B200_DEBUG", 0),
                       env_int("MI_B200_FIXED", 1), env_int("MI_B200_TABLE_THR", 4096),
                       env_int("MI_B200_PACE", -1), env_int("MI_B200_TAIL", 1), env_int("MI_B200_FP4", 1),
                       env_int("MI_B200_EVAC", 1), env_int("MI_B200_SHARD", 1),
                       env_int("MI_B200_HYBRID", 0), env_int("MI_B200_UNPERM_CTAS", 0),
                       env_int("MI_B200_INGEST", 4), env_int("MI_B200_INGEST_SPLIT", 0),
                       env_int("MI_B200_SERP", 1), env_int("MI_B200_F32_EPI", 1), env_int("MI_B200_XP", -1),
                       env_int("MI_B200_XP_COLS", 3072), env_int("MI_B200_XP_STATS", 1),
                       env_int("MI_B200_XP_DIAG_W", 90)};
    return t;
}
int cta_group() { return tuning().cta_group; }
// Operand format: e2m1 nibbles for kind::mxf4 (twice the int8 MMA rate, half
// the bytes) on SM pairs while fp32 accumulation is exact (N < 2^24), else
// int8.  mi_unpack_colsum and mi_gram_mi both follow this rule, so the knob
// must not change between them.
bool operand_fp4(int64_t n_rows) { return tuning().fp4 && tuning().cta_group == 2 && n_rows < kFp4MaxN; }
// The word-operand build (expansion inside the GEMM's producer, no X in HBM)
// where writing and re-reading X costs a large share of the step: narrow m
// (the unpack is O(N m), the GEMM O(N m^2)).  Knob "xp": -1 auto (m_pad <=
// "xp_cols", a third of it for odd word counts), 0 never, 1 whenever the
// operands are e2m1.
bool words_operand(int64_t n_rows, int64_t n_cols) {
    const Tuning& t = tuning();
    if (!operand_fp4(n_rows) || t.xp == 0) return false;
    // an odd word count per column costs the build a padded copy of the words
    // (its TMA map needs a 16-byte row pitch): N = 8e6 + 64, m = 512 steps
    // 0.87 ms against 0.52 ms with an even count and 0.94 ms on the unpack
    // path; at m = 2048 the two paths tie.  So the limit is a third of xp_cols.
    const bool odd = ((n_rows + 63) / 64) % 2 != 0;
    return t.xp == 1 || round_up(n_cols < 1 ? 1 : n_cols, 256) <= (odd ? t.xp_cols / 3 : t.xp_cols);
}
int prefetch_dist() { return tuning().prefetch; }
int l2_hint() { return tuning().l2_hint; }
int tile_band() { return tuning().band > 0 ? tuning().band : 8; }

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }


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

}  // namespace capi
}  // namespace mib200

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

int mi_words_operand(int64_t n_rows, int64_t n_cols) { return words_operand(n_rows, n_cols) ? 1 : 0; }

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
        if (value < 0 || value > 4) return fail(MI_ERR_DOMAIN, "l2_hint must be 0 .. 4");
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
    } else if (!strcmp(key, "debug")) {  // experiments only (GramMiParams::debug bit mask)
        t.debug = value;
    } else if (!strcmp(key, "xp")) {
        if (value < -1 || value > 1) return fail(MI_ERR_DOMAIN, "xp must be -1 (auto), 0 (off) or 1 (on)");
        t.xp = value;
    } else if (!strcmp(key, "xp_stats")) {
        if (value != 0 && value != 1) return fail(MI_ERR_DOMAIN, "xp_stats must be 0 or 1");
        t.xp_stats = value;
    } else if (!strcmp(key, "xp_diag_w")) {
        if (value < 10 || value > 100) return fail(MI_ERR_DOMAIN, "xp_diag_w must be in [10, 100] (percent)");
        t.xp_diag_w = value;
    } else if (!strcmp(key, "xp_cols")) {
        if (value < 0) return fail(MI_ERR_DOMAIN, "xp_cols must be >= 0");
        t.xp_cols = value;
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
    if (!strcmp(key, "xp")) return t.xp;
    if (!strcmp(key, "debug")) return t.debug;
    if (!strcmp(key, "xp_cols")) return t.xp_cols;
    if (!strcmp(key, "xp_diag_w")) return t.xp_diag_w;
    if (!strcmp(key, "xp_stats")) return t.xp_stats;
    return -1;
}

}  // extern "C"
