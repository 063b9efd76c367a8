// Internal interface shared by the C-ABI translation units (capi_common.cu,
// dealing.cu, launch.cu, host_path.cu, bmi.cu).  Nothing here is exported in
// include/mimatrix_b200.h.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "mi_kernels.h"

namespace mib200 {
namespace capi {

// ---- error state (thread-local message behind mi_last_error)
extern thread_local char g_err[512];
int fail(int code, const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);

#define MI_CUDA(call)                                              \
    do {                                                           \
        cudaError_t e_ = (call);                                   \
        if (e_ != cudaSuccess) return ::mib200::capi::cuda_fail(e_, #call); \
    } while (0)

// ---- tuning knobs (mi_set_tuning / MI_B200_* env)
constexpr int kMaxIngestStages = 16;
int env_int(const char* name, int dflt);
struct Tuning {
    int cta_group, prefetch, l2_hint, band, stages, epi_warps, debug, fixed, table_thr, pace, tail, fp4, evac, shard,
        hybrid, unperm_ctas, ingest, ingest_split, serp, f32_epi, xp, xp_cols, xp_stats, xp_diag_w;
};
// the word-operand build (mi_words_operand's rule)
bool words_operand(int64_t n_rows, int64_t n_cols);
Tuning& tuning();
int cta_group();
bool operand_fp4(int64_t n_rows);
int prefetch_dist();
int l2_hint();
int tile_band();

// ---- devices
struct DevInfo {
    int num_sms = 0;
    int major = 0;
    int minor = 0;
};
int query_device(int device, DevInfo* out);
int current_device_info(DevInfo* out);

// ---- layout of the colstat workspace and argument checks
int64_t round_up(int64_t x, int64_t a);
long long* xlogx_ptr(void* colstat, int64_t n_rows, int64_t n_cols);
int2* blkrange_ptr(void* colstat, int64_t n_rows, int64_t n_cols);
float* fixr_ptr(void* colstat, int64_t n_rows, int64_t n_cols);
int check_shape(int64_t n_rows, int64_t n_cols);
int check_mode(int mode, double eps, int out_kind);
int check_padding(const uint64_t* h_words, int64_t n_rows, int64_t n_cols);

// ---- tile dealing (dealing.cu)
int64_t tiles_per_side(int64_t n_cols);
std::vector<int32_t> all_tiles(int64_t T, int band, int first = 0);
std::vector<int32_t> rank_tiles(int64_t T, int rank, int world, int band);

// ---- the fused kernel launch (launch.cu); tail plan shared with the host path
struct TailPlan {
    int n_full, split, kmode, epi;
    int units;                        // sum of cnt
    unsigned char cnt[kTailMaxUnits];  // units of tail tile i
};
TailPlan tail_plan(int64_t n_tiles, int cg, int clusters, int nkb, const int32_t* h_tiles = nullptr, int diag_w = 100,
                   int epi_parts = 2);
int tail_epi_parts(bool xp);  // epilogue warps per TMEM lane quadrant of the build
int launch_fused(const int8_t* d_kmajor, const void* d_colstat, int64_t n_rows, int64_t n_cols, int64_t ld, int mode,
                 double epsilon, int include_diagonal, int out_kind, void* d_out, int64_t ld_out, const int32_t* d_tiles,
                 int64_t n_tiles, unsigned int* row_done, cudaStream_t stream, const uint64_t* d_words = nullptr,
                 bool stats = false, int32_t* d_colsum = nullptr);

}  // namespace capi
}  // namespace mib200
