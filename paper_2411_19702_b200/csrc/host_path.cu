// Host-buffer entry points (mi_all_pairs_host and friends): the cached
// per-device workspace, pinned staging of pageable words with host copy
// threads, the staged upload -> unpack -> compute -> download pipeline, the
// row-band egress that overlaps the fused kernel, and the sharded egress.
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
#include <string>
#include <vector>

#include "../../include/mimatrix_b200.h"
#include "capi_internal.h"
#include "mi_kernels.h"
#include "milog.cuh"

using namespace mib200;
using namespace mib200::capi;

namespace mib200 {
namespace capi {

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
    void* h_egress = nullptr; size_t h_egress_cap = 0;  // pinned staging of a pageable host output
    std::vector<cudaEvent_t> piece_ev;  // staged path: one per D2H piece (pageable output)
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
    if (w.h_egress) cudaFreeHost(w.h_egress), w.h_egress = nullptr;
    w.h_egress_cap = 0;
    for (auto& e : w.piece_ev)
        if (e) cudaEventDestroy(e);
    w.piece_ev.clear();
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

// Host threads copying between pageable user memory and pinned buffers: one
// per core up to 16 (MI_B200_COPY_THREADS overrides).  A fresh output's first
// touch (page faults) rides on these copies: config 3's drop-in takes 45.5 ms
// with 8 threads and 38.4 ms with 16 on the 16-core host (tools/dropin_e2e.py).
int copy_threads_default() {
    const int hw = (int)std::thread::hardware_concurrency();
    return std::max(1, std::min(16, env_int("MI_B200_COPY_THREADS", hw > 0 ? hw : 8)));
}

// Host copy threads between pageable user memory and the pinned staging
// buffers: one thread reaches ~10 GB/s, well short of the link's ~55.  The
// workers are a small persistent pool (created on first use, never torn
// down: spawning 8 threads per group cost ~1 ms a call); one batch at a time.
struct CopyPool {
    std::mutex mu;
    std::condition_variable cv, done_cv;
    std::vector<std::thread> workers;
    // rows x width bytes, row r from src + r spitch to dst + r dpitch
    struct Job { char* dst; const char* src; size_t width, rows, dpitch, spitch; };
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
                    if (j.rows == 1 || (j.dpitch == j.width && j.spitch == j.width))
                        memcpy(j.dst, j.src, j.width * j.rows);
                    else
                        for (size_t r = 0; r < j.rows; ++r) memcpy(j.dst + r * j.dpitch, j.src + r * j.spitch, j.width);
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
std::mutex g_copy_mu;  // one batch at a time (callers on several device threads take turns)

// 2-D copy (rows of `width` bytes) split over up to `threads` host threads.
void parallel_copy_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows,
                      int threads) {
    if (!rows || !width) return;
    const size_t bytes = width * rows;
    const size_t min_chunk = (size_t)4 << 20;
    const int t = (int)std::min<size_t>(std::min<size_t>((size_t)threads, rows), (bytes + min_chunk - 1) / min_chunk);
    if (t <= 1) {
        for (size_t r = 0; r < rows; ++r) memcpy((char*)dst + r * dpitch, (const char*)src + r * spitch, width);
        return;
    }
    std::lock_guard<std::mutex> serial(g_copy_mu);
    CopyPool& pool = copy_pool();
    pool.ensure(t);
    const size_t per = (rows + t - 1) / t;
    {
        std::lock_guard<std::mutex> lk(pool.mu);
        pool.jobs.clear();
        pool.next = 0;
        for (size_t r0 = 0; r0 < rows; r0 += per)
            pool.jobs.push_back({(char*)dst + r0 * dpitch, (const char*)src + r0 * spitch, width,
                                 std::min(per, rows - r0), dpitch, spitch});
        pool.pending = pool.jobs.size();
    }
    pool.cv.notify_all();
    std::unique_lock<std::mutex> lk(pool.mu);
    pool.done_cv.wait(lk, [&] { return pool.pending == 0; });
}

// memcpy with up to `threads` host threads.
void parallel_memcpy(void* dst, const void* src, size_t bytes, int threads) {
    const size_t chunk = (size_t)1 << 20;  // as 1 MB rows, split over the threads
    const size_t rows = bytes / chunk;
    if (rows) parallel_copy_2d(dst, chunk, src, chunk, chunk, rows, threads);
    if (bytes % chunk) memcpy((char*)dst + rows * chunk, (const char*)src + rows * chunk, bytes % chunk);
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
    const int threads = copy_threads_default();
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

// Pageable host outputs (the drop-in's fresh numpy array) are filled through
// a cached pinned egress buffer of the output's size: the copy engine writes
// it at link speed and host threads copy each finished piece out while the
// next pieces are still in flight (the driver's own pageable D2H runs at
// ~10 GB/s).  Grow-only; released by mi_release_workspace.
int egress_buffer(Workspace& ws, size_t bytes, void** out) {
    if (ws.h_egress_cap < bytes) {
        if (ws.h_egress) cudaFreeHost(ws.h_egress);
        ws.h_egress = nullptr;
        ws.h_egress_cap = 0;
        MI_CUDA(cudaHostAlloc(&ws.h_egress, bytes, cudaHostAllocDefault));
        ws.h_egress_cap = bytes;
    }
    *out = ws.h_egress;
    return MI_OK;
}

// defer_stats: on the word-operand path leave the column statistics to
// run_fused (computed inside the fused launch); otherwise kernel 1 does them.
int stage_inputs(Workspace& ws, const uint64_t* h_words, int64_t n_rows, int64_t n_cols, int64_t* ld_out,
                 int64_t* m_pad_out, const DevInfo& info, bool defer_stats = false) {
    const int64_t nw = (n_rows + 63) / 64;
    const int64_t ld = mi_kmajor_ld(n_rows);
    const int64_t m_pad = mi_kmajor_rows(n_cols);
    int rc;
    // the word-operand build needs no X: kernel 1 only counts (x = nullptr)
    const bool xp = words_operand(n_rows, n_cols);
    if ((rc = ensure(&ws.words, &ws.words_cap, (size_t)(n_cols * nw * 8)))) return rc;
    if (!xp && (rc = ensure(&ws.x, &ws.x_cap, (size_t)(m_pad * ld)))) return rc;
    if ((rc = ensure(&ws.colsum, &ws.colsum_cap, (size_t)(m_pad * 4)))) return rc;
    if ((rc = ensure(&ws.colstat, &ws.colstat_cap, (size_t)mi_colstat_bytes(n_rows, n_cols)))) return rc;
    if ((rc = upload_words(ws, h_words, n_cols, nw))) return rc;
    *ld_out = ld;
    *m_pad_out = m_pad;
    if (xp && defer_stats) return MI_OK;  // the word-operand launch computes them (run_fused)
    MI_CUDA(launch_unpack_colsum((const uint64_t*)ws.words, n_rows, n_cols, nw, xp ? nullptr : (int8_t*)ws.x, ld, m_pad,
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

// stats: the inputs were staged with defer_stats (word-operand path: the
// launch computes the column statistics too)
int run_fused(Workspace& ws, int64_t n_rows, int64_t n_cols, int64_t ld, int64_t m_pad, int mode, double eps,
              int include_diagonal, int out_kind, void* d_out, int64_t ld_out, const DevInfo& info,
              unsigned int* row_done = nullptr, bool stats = false) {
    (void)m_pad;
    const int64_t n_tiles = mi_num_tiles(n_cols);
    std::vector<int32_t> tiles = all_tiles(tiles_per_side(n_cols), tile_band(), row_done ? 1 : 0);
    int rc;
    if ((rc = ensure(&ws.tiles, &ws.tiles_cap, tiles.size() * 4))) return rc;
    MI_CUDA(cudaMemcpyAsync(ws.tiles, tiles.data(), tiles.size() * 4, cudaMemcpyHostToDevice, ws.stream));
    (void)info;
    const bool xp = words_operand(n_rows, n_cols);
    return launch_fused(xp ? nullptr : (const int8_t*)ws.x, ws.colstat, n_rows, n_cols, ld, mode, eps, include_diagonal,
                        out_kind, d_out, ld_out, (const int32_t*)ws.tiles, n_tiles, row_done, ws.stream,
                        xp ? (const uint64_t*)ws.words : nullptr, xp && stats, xp ? (int32_t*)ws.colsum : nullptr);
}

}  // namespace capi
}  // namespace mib200

extern "C" {

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
    const bool xp = words_operand(n_rows, n_cols);  // no X: the GEMM expands the words itself
    if ((rc = ensure(&ws.words, &ws.words_cap, (size_t)(n_cols * nw * 8)))) return rc;
    if (!xp && (rc = ensure(&ws.x, &ws.x_cap, (size_t)(m_pad * ld)))) return rc;
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
    const int copy_threads = copy_threads_default();
    // pageable output: D2H into the pinned egress buffer, pieces copied out below
    const bool stage_out = !host_is_pinned(h_out);
    char* d2h_dst = (char*)h_out;
    if (stage_out) {
        void* eb = nullptr;
        if ((rc = egress_buffer(ws, (size_t)n_cols * (size_t)n_cols * esz, &eb))) return rc;
        d2h_dst = (char*)eb;
    }
    struct Piece { int64_t r0, rows, c0, cols; };
    std::vector<Piece> pieces;
    auto piece_done = [&](const Piece& pc) -> int {  // record the piece's completion on the copy stream
        if (!stage_out) return MI_OK;
        const size_t k = pieces.size();
        if (ws.piece_ev.size() <= k) {
            cudaEvent_t e;
            MI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ws.piece_ev.push_back(e);
        }
        MI_CUDA(cudaEventRecord(ws.piece_ev[k], ws.copy_stream));
        pieces.push_back(pc);
        return MI_OK;
    };
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
        MI_CUDA(launch_unpack_range((const uint64_t*)ws.words, n_rows, n_cols, nw, xp ? nullptr : (int8_t*)ws.x, ld,
                                    m_pad, (int32_t*)ws.colsum, cs, xl ? br : nullptr, fp4, nullptr, tile,
                                    blk[g] * tile, u1, info.num_sms, ws.stream));
        if ((rc = launch_fused(xp ? nullptr : (const int8_t*)ws.x, ws.colstat, n_rows, n_cols, ld, mode, epsilon,
                               include_diagonal, out_kind, ws.out, n_cols, (const int32_t*)ws.tiles + 2 * first[g],
                               first[g + 1] - first[g], nullptr, ws.stream, xp ? (const uint64_t*)ws.words : nullptr)))
            return rc;
        MI_CUDA(cudaEventRecord(ws.stage_ev[g], ws.stream));
        mark(ws.stream);  // compute g done
        MI_CUDA(cudaStreamWaitEvent(ws.copy_stream, ws.stage_ev[g], 0));
        mark(ws.copy_stream);  // D2H g may start
        char* ho = d2h_dst;
        const char* dv = (const char*)ws.out;
        if (c0 > 0 && c1 > c0) {  // rows above the group, the group's columns
            MI_CUDA(cudaMemcpy2DAsync(ho + c0 * esz, pitch, dv + c0 * esz, pitch, (size_t)(c1 - c0) * esz,
                                      (size_t)c0, cudaMemcpyDeviceToHost, ws.copy_stream));
            if ((rc = piece_done({0, c0, c0, c1 - c0}))) return rc;
        }
        // the group's rows, columns [0, c1); one linear copy when they are whole
        // rows (the last group): 2-D copies run at ~52 GB/s against ~57 GB/s
        // linear on this link (tools/d2h_2d.py).  With a pageable output the
        // last rows go in 4 pieces, so the host copies trail the link closely.
        if (c1 > c0 && c1 == n_cols) {
            const int64_t parts = stage_out ? std::min<int64_t>(4, c1 - c0) : 1;
            for (int64_t q = 0; q < parts; ++q) {
                const int64_t a = c0 + (c1 - c0) * q / parts, b = c0 + (c1 - c0) * (q + 1) / parts;
                if (b <= a) continue;
                MI_CUDA(cudaMemcpyAsync(ho + a * pitch, dv + a * pitch, (size_t)(b - a) * pitch,
                                        cudaMemcpyDeviceToHost, ws.copy_stream));
                if ((rc = piece_done({a, b - a, 0, n_cols}))) return rc;
            }
        } else if (c1 > c0) {
            MI_CUDA(cudaMemcpy2DAsync(ho + c0 * pitch, pitch, dv + c0 * pitch, pitch, (size_t)c1 * esz,
                                      (size_t)(c1 - c0), cudaMemcpyDeviceToHost, ws.copy_stream));
            if ((rc = piece_done({c0, c1 - c0, 0, c1}))) return rc;
        }
        mark(ws.copy_stream);  // D2H g done
    }
    // pageable output: copy each piece out as soon as its D2H has landed
    for (size_t k = 0; k < pieces.size(); ++k) {
        MI_CUDA(cudaEventSynchronize(ws.piece_ev[k]));
        const Piece& pc = pieces[k];
        const size_t off = ((size_t)pc.r0 * (size_t)n_cols + (size_t)pc.c0) * esz;
        parallel_copy_2d((char*)h_out + off, pitch, d2h_dst + off, pitch, (size_t)pc.cols * esz, (size_t)pc.rows,
                         copy_threads);
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
    if ((rc = stage_inputs(*ws, h_words, n_rows, n_cols, &ld, &m_pad, info, true))) return rc;
    stamp("H2D + unpack enqueued");
    const size_t esz = out_kind == MI_OUT_F64 ? 8 : 4;
    const size_t row_bytes = (size_t)n_cols * esz;
    // byte offset of row r's first element in the output (full or packed upper triangle)
    auto row_off = [&](int64_t r) -> size_t {
        return packed ? (size_t)(r * n_cols - (r * (r - 1)) / 2) * esz : (size_t)r * row_bytes;
    };
    if ((rc = ensure(&ws->out, &ws->out_cap, row_off(n_cols)))) return rc;
    // pageable output: D2H into the pinned egress buffer, one host copy at the end
    const bool stage_out = !host_is_pinned(h_out);
    char* d2h_dst = (char*)h_out;
    if (stage_out) {
        void* eb = nullptr;
        if ((rc = egress_buffer(*ws, row_off(n_cols), &eb))) return rc;
        d2h_dst = (char*)eb;
    }
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
        const TailPlan tp = tail_plan(nt, (int)cg, info.num_sms / (int)cg, (int)(mi_kmajor_ld(n_rows) / 128), tl.data(),
                                      words_operand(n_rows, n_cols) ? tuning().xp_diag_w : 100,
                                      tail_epi_parts(words_operand(n_rows, n_cols)));
        for (int64_t k = 0; k < nt; ++k) expect[(size_t)tl[2 * k]] += cg * (k >= tp.n_full ? (unsigned)tp.epi : 1u);
    }
    if ((rc = run_fused(*ws, n_rows, n_cols, ld, m_pad, mode, epsilon, include_diagonal, out_kind, ws->out,
                        packed ? MI_PACKED_UPPER : n_cols, info, ws->row_done_d, true)))
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
            MI_CUDA(cudaMemcpyAsync(d2h_dst + row_off(copied), (char*)ws->out + row_off(copied),
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
    if (stage_out)
        parallel_memcpy(h_out, d2h_dst, row_off(n_cols), copy_threads_default());
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
    if ((rc = stage_inputs(*ws, h_words, n_rows, n_cols, &ld, &m_pad, info, true))) return rc;
    const size_t out_bytes = (size_t)n_cols * (size_t)n_cols * 4;
    if ((rc = ensure(&ws->out, &ws->out_cap, out_bytes))) return rc;
    if ((rc = run_fused(*ws, n_rows, n_cols, ld, m_pad, MI_MODE_EXACT, 1e-12, 1, MI_OUT_COUNTS, ws->out, n_cols,
                        info, nullptr, true)))
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
    MI_CUDA(cudaHostRegister(h_ptr, (size_t)bytes, cudaHostRegisterPortable | cudaHostRegisterMapped));
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

}  // extern "C"

// ---------------------------------------------------------------- several devices, one process
//
// mi_all_pairs_host over a list of devices: the upper-triangle tiles are dealt
// as over the ranks of the multi-GPU path (mi_tile_list / mi_rank_blocks for
// rank r of world n), each device uploads the words over its own link, unpacks
// only its column blocks (the word-operand build: counts only), computes its
// tiles tile-major, and writes its tiles and mirrors straight into the mapped
// host matrix (mi_scatter_tiles' zero-copy kernel) over its own link.  One host
// thread per device.  A device may be listed twice (tests run [0, 0] on one GPU).
namespace mib200 {
namespace capi {

constexpr int kMaxSlots = 16;
Workspace g_ws_slot[kMaxSlots];
std::mutex g_multi_mu;
void* g_multi_stage = nullptr;  // pinned (portable) copy of pageable words
size_t g_multi_stage_cap = 0;
void* g_multi_egress = nullptr;  // pinned, mapped, portable matrix for a pageable output
size_t g_multi_egress_cap = 0;

int grow_pinned(void** p, size_t* cap, size_t need, unsigned flags) {
    if (*cap >= need && *p) return MI_OK;
    if (*p) cudaFreeHost(*p);
    *p = nullptr;
    *cap = 0;
    MI_CUDA(cudaHostAlloc(p, need, flags));
    *cap = need;
    return MI_OK;
}

int multi_slot(int slot, int device, const uint64_t* src_words, int64_t n_rows, int64_t n_cols, int world, int mode,
               double eps, int include_diagonal, int out_kind, void* h_dst) {
    MI_CUDA(cudaSetDevice(device));
    DevInfo info;
    int rc = query_device(device, &info);
    if (rc) return rc;
    Workspace& ws = g_ws_slot[slot];
    if (ws.device != device) release(ws);
    if (ws.device < 0) {
        ws.device = device;
        MI_CUDA(cudaStreamCreateWithFlags(&ws.stream, cudaStreamNonBlocking));
        MI_CUDA(cudaStreamCreateWithFlags(&ws.copy_stream, cudaStreamNonBlocking));
    }
    const int64_t T = tiles_per_side(n_cols);
    const std::vector<int32_t> tiles = rank_tiles(T, slot, world, tile_band());
    const int64_t k = (int64_t)tiles.size() / 2;
    if (k == 0) return MI_OK;
    const int64_t nw = (n_rows + 63) / 64, ld = mi_kmajor_ld(n_rows), m_pad = mi_kmajor_rows(n_cols);
    const int ts = mi_tile_size();
    const size_t esz = out_kind == MI_OUT_F64 ? 8 : 4;
    const bool xp = words_operand(n_rows, n_cols);
    if ((rc = ensure(&ws.words, &ws.words_cap, (size_t)(n_cols * nw * 8)))) return rc;
    if (!xp && (rc = ensure(&ws.x, &ws.x_cap, (size_t)(m_pad * ld)))) return rc;
    if ((rc = ensure(&ws.colsum, &ws.colsum_cap, (size_t)(m_pad * 4 + T)))) return rc;  // + the block mask
    if ((rc = ensure(&ws.colstat, &ws.colstat_cap, (size_t)mi_colstat_bytes(n_rows, n_cols)))) return rc;
    if ((rc = ensure(&ws.tiles, &ws.tiles_cap, tiles.size() * 4))) return rc;
    if ((rc = ensure(&ws.out, &ws.out_cap, (size_t)k * ts * ts * esz))) return rc;
    MI_CUDA(cudaMemcpyAsync(ws.words, src_words, (size_t)(n_cols * nw * 8), cudaMemcpyHostToDevice, ws.stream));
    MI_CUDA(cudaMemcpyAsync(ws.tiles, tiles.data(), tiles.size() * 4, cudaMemcpyHostToDevice, ws.stream));
    uint8_t* d_mask = nullptr;
    if (!xp) {  // expand only this slot's column blocks
        std::vector<uint8_t> mask((size_t)T, 0);
        const int64_t got = mi_rank_blocks(n_cols, slot, world, mask.data(), T);
        if (got < 0) return (int)-got;
        d_mask = (uint8_t*)ws.colsum + m_pad * 4;
        MI_CUDA(cudaMemcpyAsync(d_mask, mask.data(), (size_t)T, cudaMemcpyHostToDevice, ws.stream));
    }
    MI_CUDA(launch_unpack_colsum((const uint64_t*)ws.words, n_rows, n_cols, nw, xp ? nullptr : (int8_t*)ws.x, ld, m_pad,
                                 (int32_t*)ws.colsum, (ColStat*)ws.colstat, xlogx_ptr(ws.colstat, n_rows, n_cols),
                                 blkrange_ptr(ws.colstat, n_rows, n_cols), fixr_ptr(ws.colstat, n_rows, n_cols),
                                 operand_fp4(n_rows), d_mask, ts, info.num_sms, ws.stream));
    if ((rc = launch_fused(xp ? nullptr : (const int8_t*)ws.x, ws.colstat, n_rows, n_cols, ld, mode, eps,
                           include_diagonal, out_kind, ws.out, MI_TILE_MAJOR, (const int32_t*)ws.tiles, k, nullptr,
                           ws.stream, xp ? (const uint64_t*)ws.words : nullptr)))
        return rc;
    void* d_dst = nullptr;  // the mapped host matrix as this device sees it
    MI_CUDA(cudaHostGetDevicePointer(&d_dst, h_dst, 0));
    MI_CUDA(launch_scatter_tiles(ws.out, (const int32_t*)ws.tiles, k, ts, n_cols, (int)esz, d_dst, n_cols, true,
                                 ws.stream));
    MI_CUDA(cudaStreamSynchronize(ws.stream));
    return MI_OK;
}

}  // namespace capi
}  // namespace mib200

extern "C" {

int mi_all_pairs_host_devices(const uint64_t* h_words, int64_t n_rows, int64_t n_cols, int mode, double epsilon,
                              int include_diagonal, int out_kind, void* h_out, const int* devices, int n_devices) {
    int rc = check_shape(n_rows, n_cols);
    if (rc) return rc;
    if ((rc = check_mode(mode, epsilon, out_kind))) return rc;
    if (out_kind == MI_OUT_COUNTS) return fail(MI_ERR_DOMAIN, "use mi_gram_ones_host for counts");
    if (!devices || n_devices < 1 || n_devices > kMaxSlots)
        return fail(MI_ERR_DOMAIN, "devices must list 1..%d device indices", kMaxSlots);
    if (n_devices == 1)
        return mi_all_pairs_host(h_words, n_rows, n_cols, mode, epsilon, include_diagonal, out_kind, h_out, devices[0]);
    if ((rc = check_padding(h_words, n_rows, n_cols))) return rc;
    for (int r = 0; r < n_devices; ++r) {
        DevInfo info;
        if ((rc = query_device(devices[r], &info))) return rc;
    }
    std::lock_guard<std::mutex> lk(g_multi_mu);
    const int64_t nw = (n_rows + 63) / 64;
    const size_t words_bytes = (size_t)(n_cols * nw * 8);
    const size_t out_bytes = (size_t)n_cols * (size_t)n_cols * (out_kind == MI_OUT_F64 ? 8 : 4);
    const int threads = copy_threads_default();
    // inputs every device can DMA from: the caller's pinned words, or a portable pinned copy
    const uint64_t* src = h_words;
    if (!host_is_pinned(h_words)) {
        if ((rc = grow_pinned(&g_multi_stage, &g_multi_stage_cap, words_bytes, cudaHostAllocPortable))) return rc;
        parallel_memcpy(g_multi_stage, h_words, words_bytes, threads);
        src = (const uint64_t*)g_multi_stage;
    }
    // output every device can write: the caller's mapped pinned matrix, or a cached one copied out at the end
    void* dst = h_out;
    cudaPointerAttributes a;
    const bool mapped = cudaPointerGetAttributes(&a, h_out) == cudaSuccess && a.type == cudaMemoryTypeHost &&
                        a.devicePointer != nullptr;
    cudaGetLastError();
    if (!mapped) {
        if ((rc = grow_pinned(&g_multi_egress, &g_multi_egress_cap, out_bytes,
                              cudaHostAllocPortable | cudaHostAllocMapped)))
            return rc;
        dst = g_multi_egress;
    }
    std::vector<int> rcs((size_t)n_devices, MI_OK);
    std::vector<std::string> msgs((size_t)n_devices);
    std::vector<std::thread> pool;
    for (int r = 0; r < n_devices; ++r)
        pool.emplace_back([&, r] {
            rcs[(size_t)r] = multi_slot(r, devices[r], src, n_rows, n_cols, n_devices, mode, epsilon,
                                        include_diagonal, out_kind, dst);
            if (rcs[(size_t)r]) msgs[(size_t)r] = mi_last_error();
        });
    for (auto& t : pool) t.join();
    for (int r = 0; r < n_devices; ++r)
        if (rcs[(size_t)r]) return fail(rcs[(size_t)r], "device %d: %s", devices[r], msgs[(size_t)r].c_str());
    if (!mapped) parallel_memcpy(h_out, dst, out_bytes, threads);
    return MI_OK;
}

void mi_release_workspace(void) {
    {
        std::lock_guard<std::mutex> lk(g_ws_mu);
        for (auto& w : g_ws) release(w);
    }
    std::lock_guard<std::mutex> lk(g_multi_mu);
    for (auto& w : g_ws_slot) release(w);
    if (g_multi_stage) cudaFreeHost(g_multi_stage), g_multi_stage = nullptr, g_multi_stage_cap = 0;
    if (g_multi_egress) cudaFreeHost(g_multi_egress), g_multi_egress = nullptr, g_multi_egress_cap = 0;
}

}  // extern "C"
