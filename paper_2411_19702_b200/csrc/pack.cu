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

constexpr int kPackWordsPerThread = 4;  // 256 rows

__global__ void __launch_bounds__(256) pack_bits_kernel(const uint8_t* __restrict__ bits, int64_t n_rows, int64_t m,
                                                         int64_t ld, uint64_t* __restrict__ words, int64_t nw,
                                                         int* __restrict__ bad) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // column group
    const int64_t c8 = g * 8;
    if (c8 >= m) return;
    const bool full8 = c8 + 8 <= m && (ld % 8 == 0) && ((reinterpret_cast<uintptr_t>(bits) & 7) == 0);
    const int64_t ny = (nw + kPackWordsPerThread - 1) / kPackWordsPerThread;
    uint64_t badv = 0;
    for (int64_t y = blockIdx.y; y < ny; y += gridDim.y) {
        const int64_t w0 = y * kPackWordsPerThread;
        uint64_t out[8][kPackWordsPerThread];
#pragma unroll
        for (int q = 0; q < kPackWordsPerThread; ++q) {
            uint64_t X[8];
#pragma unroll
            for (int gq = 0; gq < 8; ++gq) {
                uint64_t v[8];
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const int64_t row = (w0 + q) * 64 + gq * 8 + r;
                    const uint8_t* src = bits + row * ld + c8;
                    if (row >= n_rows) {
                        v[r] = 0;
                    } else if (full8) {
                        v[r] = __ldcs(reinterpret_cast<const unsigned long long*>(src));
                    } else {
                        uint64_t x = 0;
                        for (int j = 0; j < 8; ++j)
                            if (c8 + j < m) x |= (uint64_t)src[j] << (8 * j);
                        v[r] = x;
                    }
                }
                uint64_t x = 0;
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    badv |= v[r];
                    x |= (v[r] & 0x0101010101010101ull) << r;
                }
                X[gq] = x;  // byte j = column c8 + j, rows 8 gq .. 8 gq + 7
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                uint64_t w = 0;
#pragma unroll
                for (int gq = 0; gq < 8; ++gq) w |= ((X[gq] >> (8 * j)) & 0xFFull) << (8 * gq);
                out[j][q] = w;
            }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (c8 + j >= m) break;
            uint64_t* dst = words + (c8 + j) * nw + w0;
            if (w0 + kPackWordsPerThread <= nw && (reinterpret_cast<uintptr_t>(dst) & 31) == 0) {
                asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(dst), "l"(out[j][0]), "l"(out[j][1]),
                             "l"(out[j][2]), "l"(out[j][3])
                             : "memory");
            } else {
#pragma unroll
                for (int q = 0; q < kPackWordsPerThread; ++q)
                    if (w0 + q < nw) dst[q] = out[j][q];
            }
        }
    }
    if (badv & 0xFEFEFEFEFEFEFEFEull) atomicOr(bad, 1);
}

cudaError_t launch_pack_bits(const uint8_t* bits, int64_t n_rows, int64_t m, int64_t ld, uint64_t* words, int* bad,
                             cudaStream_t stream) {
    const int64_t nw = (n_rows + 63) / 64;
    const int64_t ny = (nw + kPackWordsPerThread - 1) / kPackWordsPerThread;
    const int64_t groups = (m + 7) / 8;
    const dim3 grid((unsigned)((groups + 255) / 256), (unsigned)(ny < 65535 ? ny : 65535));
    pack_bits_kernel<<<grid, 256, 0, stream>>>(bits, n_rows, m, ld, words, nw, bad);
    return cudaGetLastError();
}

}  // namespace mib200
