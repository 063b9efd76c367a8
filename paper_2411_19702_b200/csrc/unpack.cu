// Kernel 1: bit-packed columns -> K-major int8 operand + column sums.
//
// Input is the reference's BinaryMatrix.words layout (binmat.py:3-6,57-97):
// (m, nw) uint64, column-major, bit r of word w = row 64w + r, padding zero.
// Output X holds X[c][r] = bit r of column c as 0/1 bytes in a k-blocked
// K-major layout: [ld/128 k-blocks][m_pad columns][128 bytes], so the 128 x 128
// box the GEMM loads for (k-block, 128 columns) is one contiguous 16 KB chunk
// (one DRAM page, one TLB entry).  Padding rows / columns are zero, so padded
// cells add nothing to G.
// The same pass produces v[c] = popcount of column c, i.e. the reference's
// column_sums (binmat.py:175-177), which the fused epilogue needs.
//
// HBM-bound: reads 8*m*nw bytes, writes m_pad*N_pad bytes.  One warp per
// column; each lane expands 16 bits into one 16-byte store so a warp
// instruction writes 512 contiguous bytes.
#include <cuda_runtime.h>
#include <cstdint>

#include "mi_kernels.h"
#include "milog.cuh"

namespace mib200 {

// 4 bits -> 4 bytes of 0/1 (copies of the nibble 7 bits apart never overlap,
// so the multiply places bit k at bit 8k with no carries).
__device__ __forceinline__ uint32_t spread4(uint32_t nib) { return (nib * 0x00204081u) & 0x01010101u; }

// T(c) = c log2(c) 2^s for c = 0..N with the epilogue's own fix_xlog2x, so the
// table path and the per-column terms agree bit for bit.
__global__ void __launch_bounds__(256) xlogx_table_kernel(long long* __restrict__ T, long long N, int s,
                                                          int2* __restrict__ blkrange, int nblk) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nblk; b += gridDim.x * blockDim.x)
        blkrange[b] = make_int2(0x7FFFFFFF, -1);  // (min, max) column sum, filled by the unpack
    __shared__ float R[1 << kFixLogBits];
    __shared__ float2 LG[1 << kFixLogBits];
    for (int q = threadIdx.x; q < (1 << kFixLogBits); q += blockDim.x) {
        R[q] = kFixR[q];
        LG[q] = kFixLG[q];
    }
    __syncthreads();
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c <= N; c += (long long)gridDim.x * blockDim.x)
        T[c] = fix_xlog2x((unsigned)c, s, R, LG);
}

__global__ void __launch_bounds__(256)
unpack_colsum_kernel(const uint64_t* __restrict__ words, int64_t n_rows, int64_t m, int64_t nw,
                     int8_t* __restrict__ x, int64_t ld, int64_t m_pad, int32_t* __restrict__ colsum,
                     ColStat* __restrict__ colstat, int fix_s, int2* __restrict__ blkrange) {
    const int lane = threadIdx.x & 31;
    const int quarter = lane & 3;
    const int64_t warp0 = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x / 32);
    const int64_t wpad = ld / 64;  // words per padded column
    for (int64_t c = warp0; c < m_pad; c += nwarps) {
        const uint64_t* __restrict__ src = words + c * nw;
        int8_t* __restrict__ dst = x + c * 128;  // row c inside every k-block
        const int64_t kb_stride = m_pad * 128;
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
            if (w < wpad)
                *reinterpret_cast<uint4*>(dst + (w >> 1) * kb_stride + (w & 1) * 64 + quarter * 16) = v;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (lane == 0) {
            if (colsum) colsum[c] = (int32_t)cnt;
            // marginal logs for the fused epilogue: log2(v) and log2(N - v)
            ColStat st;
            const int64_t v0 = n_rows - (int64_t)cnt;
            int e1 = 0, e0 = 0;
            st.v = (double)cnt;
            st.nv = (double)v0;
            st.f1 = cnt > 0 ? log2_frac((double)cnt, kLog2TabInit, e1) : 0.0;
            st.f0 = v0 > 0 ? log2_frac((double)v0, kLog2TabInit, e0) : 0.0;
            st.e1 = cnt > 0 ? (double)e1 : 0.0;
            st.e0 = v0 > 0 ? (double)e0 : 0.0;
            st.vi = (int)cnt;
            st.pad = 0;
            st.q = fix_xlog2x(cnt, fix_s, kFixR, kFixLG) + fix_xlog2x((unsigned)v0, fix_s, kFixR, kFixLG);
            if (blkrange && real) {
                atomicMin(&blkrange[c / 128].x, (int)cnt);
                atomicMax(&blkrange[c / 128].y, (int)cnt);
            }
            colstat[c] = st;
        }
    }
}

cudaError_t launch_unpack_colsum(const uint64_t* words, int64_t n_rows, int64_t m, int64_t nw, int8_t* x,
                                 int64_t ld, int64_t m_pad, int32_t* colsum, ColStat* colstat, long long* xlogx,
                                 int2* blkrange, int num_sms, cudaStream_t stream) {
    if (xlogx) {
        int64_t tb = (n_rows + 1 + 255) / 256;
        if (tb > (int64_t)num_sms * 16) tb = (int64_t)num_sms * 16;
        xlogx_table_kernel<<<(unsigned)tb, 256, 0, stream>>>(xlogx, n_rows, xlogx_scale(n_rows), blkrange,
                                                              blkrange ? (int)(m_pad / 128) : 0);
    }
    const int threads = 256;
    int64_t blocks = (m_pad + 7) / 8;
    const int64_t cap = (int64_t)num_sms * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    unpack_colsum_kernel<<<(unsigned)blocks, threads, 0, stream>>>(words, n_rows, m, nw, x, ld, m_pad, colsum,
                                                                   colstat, xlogx_scale(n_rows),
                                                                   xlogx ? blkrange : nullptr);
    return cudaGetLastError();
}

}  // namespace mib200
