// Device packing: a row-major uint8 0/1 matrix (N x m, the reference's
// from_bits / from_rows input, binmat.py:34-46,136-172) -> the packed words
// layout (m, nw) uint64, bit r of word w = row 64 w + r (binmat.py:3-6).
//
// No shared memory: thread (g, y) owns 8 adjacent columns 8 g .. 8 g + 7 and
// the 256 rows of words 4 y .. 4 y + 3.  It loads each row's 8 bytes as one
// uint64 (a warp reads 256 contiguous bytes of the row: coalesced; the byte
// matrix is the one large stream, so the kernel is HBM-bound on reads), and
// transposes bits in registers: for 8 rows r, X |= (v_r & 0x0101..01) << r
// puts column j's 8 bits in byte j of X; the bytes of 8 such X then assemble
// column j's 64-bit word.  ~1.5 integer ops per input byte.  The four words
// of a column go out as one 32-byte store when aligned.  A byte other than
// 0 / 1 sets *bad (from_rows's DomainError); rows >= N pack as zeros, so the
// padding bits are zero as validate_words requires.
#include <cuda_runtime.h>
#include <cstdint>

#include "mi_kernels.h"

namespace mib200 {

// 16 columns (one 16-byte load per row) x 64 rows (one word per column) per
// thread: twice the bytes per load instruction of an 8-column thread, with
// the registers of one word per column instead of four.
__global__ void __launch_bounds__(256) pack_bits_kernel(const uint8_t* __restrict__ bits, int64_t n_rows, int64_t m,
                                                         int64_t ld, uint64_t* __restrict__ words, int64_t nw,
                                                         int* __restrict__ bad) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // column group of 16
    const int64_t c16 = g * 16;
    if (c16 >= m) return;
    const bool full = c16 + 16 <= m && (ld % 16 == 0) && ((reinterpret_cast<uintptr_t>(bits) & 15) == 0);
    uint64_t badv = 0;
    for (int64_t w = blockIdx.y; w < nw; w += gridDim.y) {
        uint64_t X[8][2];  // [row group][lo / hi 8 columns]: byte j = column, bit r = row 8 gq + r
#pragma unroll
        for (int gq = 0; gq < 8; ++gq) {
            uint64_t lo[8], hi[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int64_t row = w * 64 + gq * 8 + r;
                const uint8_t* src = bits + row * ld + c16;
                if (row >= n_rows) {
                    lo[r] = hi[r] = 0;
                } else if (full) {
                    const ulonglong2 v = __ldcs(reinterpret_cast<const ulonglong2*>(src));
                    lo[r] = v.x;
                    hi[r] = v.y;
                } else {
                    uint64_t x0 = 0, x1 = 0;
                    for (int j = 0; j < 8; ++j) {
                        if (c16 + j < m) x0 |= (uint64_t)src[j] << (8 * j);
                        if (c16 + 8 + j < m) x1 |= (uint64_t)src[8 + j] << (8 * j);
                    }
                    lo[r] = x0;
                    hi[r] = x1;
                }
            }
            uint64_t x0 = 0, x1 = 0;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                badv |= lo[r] | hi[r];
                x0 |= (lo[r] & 0x0101010101010101ull) << r;
                x1 |= (hi[r] & 0x0101010101010101ull) << r;
            }
            X[gq][0] = x0;
            X[gq][1] = x1;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int64_t c = c16 + 8 * h + j;
                if (c >= m) break;
                uint64_t word = 0;
#pragma unroll
                for (int gq = 0; gq < 8; ++gq) word |= ((X[gq][h] >> (8 * j)) & 0xFFull) << (8 * gq);
                words[c * nw + w] = word;
            }
        }
    }
    if (badv & 0xFEFEFEFEFEFEFEFEull) atomicOr(bad, 1);
}

cudaError_t launch_pack_bits(const uint8_t* bits, int64_t n_rows, int64_t m, int64_t ld, uint64_t* words, int* bad,
                             cudaStream_t stream) {
    const int64_t nw = (n_rows + 63) / 64;
    const int64_t groups = (m + 15) / 16;
    const dim3 grid((unsigned)((groups + 255) / 256), (unsigned)(nw < 65535 ? nw : 65535));
    pack_bits_kernel<<<grid, 256, 0, stream>>>(bits, n_rows, m, ld, words, nw, bad);
    return cudaGetLastError();
}

// binmat.to_dense (binmat.py:187-194) for the sparse backend's data,
// SparseBinaryMatrix (per-column sorted row-index lists, binmat.py:100-133):
// the CSC index arrays -> the words layout, on the device, cost ~ nnz.  A warp
// takes 32 consecutive indices of one column (sorted, so neighbours mostly share
// a word): the lanes of each word (__match_any_sync) OR their bits together and
// one of them does the atomicOr.  An index outside [0, n_rows) sets *bad.
__global__ void __launch_bounds__(256) pack_sparse_kernel(const int64_t* __restrict__ indices,
                                                          const int64_t* __restrict__ indptr, int64_t n_rows,
                                                          int64_t m, int64_t nw, unsigned long long* __restrict__ words,
                                                          int* __restrict__ bad) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; c < m; c += warps) {
        const int64_t b = indptr[c], e = indptr[c + 1];
        for (int64_t i0 = b; i0 < e; i0 += 32) {
            const int64_t i = i0 + lane;
            const bool in = i < e;
            int64_t r = in ? indices[i] : 0;
            if (in && (r < 0 || r >= n_rows)) {
                atomicOr(bad, 1);
                r = 0;
            }
            const unsigned act = __ballot_sync(0xffffffffu, in);
            const long long w = in ? r >> 6 : -1 - lane;  // idle lanes never match a word
            const unsigned grp = __match_any_sync(0xffffffffu, w);
            const unsigned long long bit = in ? 1ull << (r & 63) : 0ull;
            // OR of the group's bits: 64-bit as two 32-bit reductions
            const unsigned lo = __reduce_or_sync(grp, (unsigned)bit), hi = __reduce_or_sync(grp, (unsigned)(bit >> 32));
            if (in && lane == __ffs(grp & act) - 1)
                atomicOr(words + c * nw + w, ((unsigned long long)hi << 32) | lo);
        }
    }
}

cudaError_t launch_pack_sparse(const int64_t* indices, const int64_t* indptr, int64_t n_rows, int64_t m,
                               uint64_t* words, int* bad, int num_sms, cudaStream_t stream) {
    const int64_t nw = (n_rows + 63) / 64;
    cudaError_t e = cudaMemsetAsync(words, 0, (size_t)(m * nw * 8), stream);
    if (e != cudaSuccess) return e;
    int64_t blocks = (m + 7) / 8;
    if (blocks > (int64_t)num_sms * 16) blocks = (int64_t)num_sms * 16;
    pack_sparse_kernel<<<(unsigned)blocks, 256, 0, stream>>>(indices, indptr, n_rows, m, nw,
                                                             reinterpret_cast<unsigned long long*>(words), bad);
    return cudaGetLastError();
}

// The words with a row pitch of `pitch` >= nw words (the word-operand build's
// TMA map needs a 16-byte multiple): one warp per column row and pass, 32
// consecutive words per load; the pad words are not written (TMA never reads
// them: its map's extent is nw).
__global__ void __launch_bounds__(256) pitch_words_kernel(const unsigned long long* __restrict__ src, int64_t nw,
                                                          unsigned long long* __restrict__ dst, int64_t pitch,
                                                          int64_t m) {
    // block (x, y): words [x * 2048, +2048) of columns y, y + gridDim.y, ...; 8 loads in flight per thread
    const int64_t w0 = (int64_t)blockIdx.x * 2048 + threadIdx.x;
    for (int64_t c = blockIdx.y; c < m; c += gridDim.y) {
        const unsigned long long* s = src + c * nw;
        unsigned long long* d = dst + c * pitch;
        unsigned long long v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = w0 + 256 * k < nw ? __ldcs(s + w0 + 256 * k) : 0ull;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (w0 + 256 * k < nw) d[w0 + 256 * k] = v[k];
    }
}

cudaError_t launch_pitch_words(const uint64_t* src, int64_t nw, uint64_t* dst, int64_t pitch, int64_t m, int num_sms,
                               cudaStream_t stream) {
    (void)num_sms;
    const dim3 grid((unsigned)((nw + 2047) / 2048), (unsigned)(m < 65535 ? m : 65535));
    pitch_words_kernel<<<grid, 256, 0, stream>>>(reinterpret_cast<const unsigned long long*>(src), nw,
                                                 reinterpret_cast<unsigned long long*>(dst), pitch, m);
    return cudaGetLastError();
}

}  // namespace mib200
