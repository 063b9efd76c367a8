// BMI1 ingest (the reference's packed container, io.py:92-116): header
// parsing and the payload streamed straight into device words.
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

extern "C" {


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

}  // extern "C"
