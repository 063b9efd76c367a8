// Kernel 1: bit-packed columns -> K-major int8 operand + column sums.
//
// Input is the reference's BinaryMatrix.words layout (binmat.py:3-6,57-97):
// (m, nw) uint64, column-major, bit r of word w = row 64w + r, padding zero.
// Output X[c][r] (m_pad x ld bytes, ld = N_pad % 128 == 0) holds 0/1 bytes and
// is zero in every padding row / column, so padded cells add nothing to G.
// The same pass produces v[c] = popcount of column c, i.e. the reference's
// column_sums (binmat.py:175-177), which the fused epilogue needs.
//
// HBM-bound: reads 8*m*nw bytes, writes m_pad*N_pad bytes.  One warp per
// column; each lane expands 16 bits into one 16-byte store so a warp
// instruction writes 512 contiguous bytes.
#include <cuda_runtime.h>
#include <cstdint>

#include "mi_kernels.h"

namespace mib200 {

// 4 bits -> 4 bytes of 0/1 (copies of the nibble 7 bits apart never overlap,
// so the multiply places bit k at bit 8k with no carries).
__device__ __forceinline__ uint32_t spread4(uint32_t nib) { return (nib * 0x00204081u) & 0x01010101u; }

__global__ void __launch_bounds__(256)
unpack_colsum_kernel(const uint64_t* __restrict__ words, int64_t m, int64_t nw, int8_t* __restrict__ x,
                     int64_t ld, int64_t m_pad, int32_t* __restrict__ colsum) {
    const int lane = threadIdx.x & 31;
    const int quarter = lane & 3;
    const int64_t warp0 = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x / 32);
    const int64_t wpad = ld / 64;  // words per padded column
    for (int64_t c = warp0; c < m_pad; c += nwarps) {
        const uint64_t* __restrict__ src = words + c * nw;
        uint4* __restrict__ dst = reinterpret_cast<uint4*>(x + c * ld);
        const bool real = c < m;
        uint32_t cnt = 0;
#pragma unroll 4
        for (int64_t base = 0; base < wpad; base += 8) {
            const int64_t w = base + (lane >> 2);
            const uint64_t word = (real && w < nw) ? __ldg(src + w) : 0ull;
            const uint32_t b16 = (uint32_t)(word >> (16 * quarter)) & 0xFFFFu;
            cnt += __popc(b16);
            uint4 v;
            v.x = spread4(b16 & 0xF);
            v.y = spread4((b16 >> 4) & 0xF);
            v.z = spread4((b16 >> 8) & 0xF);
            v.w = spread4(b16 >> 12);
            if (w < wpad) dst[w * 4 + quarter] = v;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (lane == 0) colsum[c] = (int32_t)cnt;
    }
}

cudaError_t launch_unpack_colsum(const uint64_t* words, int64_t m, int64_t nw, int8_t* x, int64_t ld,
                                 int64_t m_pad, int32_t* colsum, int num_sms, cudaStream_t stream) {
    const int threads = 256;
    int64_t blocks = (m_pad + 7) / 8;
    const int64_t cap = (int64_t)num_sms * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    unpack_colsum_kernel<<<(unsigned)blocks, threads, 0, stream>>>(words, m, nw, x, ld, m_pad, colsum);
    return cudaGetLastError();
}

}  // namespace mib200
