// Kernel 1: bit-packed columns -> K-major int8 operand + column sums.
//
// Input is the reference's BinaryMatrix.words layout (binmat.py:3-6,57-97):
// (m, nw) uint64, column-major, bit r of word w = row 64w + r, padding zero.
// Output X holds X[c][r] = bit r of column c as 0/1 bytes (int8 operand) or
// as e2m1 nibbles 0 / 1.0 (fp4 operand, two rows per byte) in a k-blocked
// K-major layout: [ld/128 k-blocks][m_pad columns][128 bytes], so the 128 x 128
// box the GEMM loads for (k-block, 128 columns) is one contiguous 16 KB chunk
// (one DRAM page, one TLB entry).  Padding rows / columns are zero, so padded
// cells add nothing to G.
// The same pass produces v[c] = popcount of column c, i.e. the reference's
// column_sums (binmat.py:175-177), which the fused epilogue needs.
//
// HBM-bound: reads 8*m*nw bytes, writes m_pad*N_pad (int8) or m_pad*N_pad/2
// (e2m1) bytes.  No shared memory: each thread expands whole words of one
// column straight from its loads, and a warp's stores form one contiguous run
// of X (unpack_direct_kernel, below).
#include <cuda_runtime.h>
#include <cstdint>

#include "colstat.cuh"
#include "mi_kernels.h"
#include "milog.cuh"

namespace mib200 {

// 4 bits -> 4 bytes of 0/1 (copies of the nibble 7 bits apart never overlap,
// so the multiply places bit k at bit 8k with no carries).
__device__ __forceinline__ uint32_t spread4(uint32_t nib) { return (nib * 0x00204081u) & 0x01010101u; }

// Prologue: zero the per-column count accumulators (ColStat::vi), reset the
// per-128-column (min, max) column sums, and build T(c) = c log2(c) 2^s for
// c = 0..N (when xlogx != nullptr) with the epilogue's own fix_xlog2x, so the
// table path and the per-column terms agree bit for bit.
__global__ void __launch_bounds__(256) unpack_prep_kernel(ColStat* __restrict__ colstat, int64_t m_pad,
                                                          long long* __restrict__ T, long long N, int s,
                                                          int2* __restrict__ blkrange, int nblk,
                                                          float* __restrict__ fixr) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    for (int64_t c = tid; c < m_pad; c += nthr) colstat[c].vi = 0;
    for (int64_t b = tid; b < nblk; b += nthr) blkrange[b] = make_int2(0x7FFFFFFF, -1);
    if (fixr && blockIdx.x == 0) {  // fix_xlog2x's tables for the hybrid epilogue (read through L1)
        float2* fixlg = reinterpret_cast<float2*>(fixr + (1 << kFixLogBits));
        for (int q = threadIdx.x; q < (1 << kFixLogBits); q += blockDim.x) {
            fixr[q] = kFixR[q];
            fixlg[q] = kFixLG[q];
        }
    }
    if (!T) return;
    __shared__ float R[1 << kFixLogBits];
    __shared__ float2 LG[1 << kFixLogBits];
    for (int q = threadIdx.x; q < (1 << kFixLogBits); q += blockDim.x) {
        R[q] = kFixR[q];
        LG[q] = kFixLG[q];
    }
    __syncthreads();
    for (long long c = tid; c <= N; c += nthr) T[c] = fix_xlog2x((unsigned)c, s, R, LG);
}

// Column ranges of the staged launches start on multiples of 32.
constexpr int kUnpackCols = 32;

// 64 bits -> 32 bytes of e2m1 nibbles (row 2j in the low nibble of byte j,
// row 2j + 1 in the high one; 1.0 = 0b0010), one STG.256.  fp4x8 moves bit k
// of a byte to bit 4k + 1 with three shift-or-mask steps (bits 4-7 to 16-19,
// then pairs to byte lanes, then singles to nibbles): ~8 instructions per
// byte with LOP3, half of the even/odd-split version it replaced.
__device__ __forceinline__ uint32_t fp4x8(uint32_t b) {  // b < 256
    uint32_t x = b;
    x = (x | (x << 12)) & 0x000F000Fu;
    x = (x | (x << 6)) & 0x03030303u;
    x = ((x << 1) | (x << 4)) & 0x22222222u;
    return x;
}
__device__ __forceinline__ void store_fp4_word(int8_t* dst, uint64_t w) {
    const uint32_t lo = (uint32_t)w, hi = (uint32_t)(w >> 32);
    uint32_t q[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        q[k] = fp4x8(__byte_perm(lo, 0u, 0x4440u + k));
        q[4 + k] = fp4x8(__byte_perm(hi, 0u, 0x4440u + k));
    }
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst), "r"(q[0]), "r"(q[1]),
                 "r"(q[2]), "r"(q[3]), "r"(q[4]), "r"(q[5]), "r"(q[6]), "r"(q[7])
                 : "memory");
}

// Expansion without shared memory (e2m1 case described; int8 below).  Thread (c, j) -- c one of the
// block's 64 columns (8 per warp), j = lane & 3 the word within a k-block --
// loads word 4 kb + j of column c (8 bytes: a column's four lanes read one
// full 32-byte sector) and stores its 32 bytes of nibbles with one STG.256;
// the warp's 8 columns x 128 bytes are one contiguous 1 KB run of X.  kUnr
// k-blocks are loaded before any is expanded, so every thread keeps kUnr
// loads in flight.  (The cp.async-staged kernel this replaced spent its time
// in the L1/shared pipeline at ~2.7 TB/s of writes; this box writes HBM at
// ~7 TB/s, tools/micro/write_bw.cu.)
// 64 bits -> 64 bytes of 0/1 (int8 operand): two STG.256.
__device__ __forceinline__ void store_int8_word(int8_t* dst, uint64_t w) {
    uint32_t q[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) q[k] = spread4((uint32_t)(w >> (4 * k)) & 0xFu);
#pragma unroll
    for (int h = 0; h < 2; ++h)
        asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + 32 * h),
                     "r"(q[8 * h + 0]), "r"(q[8 * h + 1]), "r"(q[8 * h + 2]), "r"(q[8 * h + 3]), "r"(q[8 * h + 4]),
                     "r"(q[8 * h + 5]), "r"(q[8 * h + 6]), "r"(q[8 * h + 7])
                     : "memory");
}

// FP4 = false: the same for the int8 operand (a 128-byte k-block row holds
// 2 words; each word becomes 64 bytes of 0/1, two STG.256), 16 columns per
// warp, so a warp's stores are one contiguous 2 KB run.
template <bool FP4>
struct DirectShape {
    static constexpr int WPK = FP4 ? 4 : 2;          // words per 128-byte k-block row
    static constexpr int COLS_PER_WARP = 32 / WPK;   // 8 (e2m1) or 16 (int8)
    static constexpr int COLS = 8 * COLS_PER_WARP;   // per 256-thread block
};
template <bool FP4, int kDirectKb, int kUnr>
__global__ void __launch_bounds__(256)
unpack_direct_kernel(const uint64_t* __restrict__ words, int64_t m, int64_t nw, int8_t* __restrict__ x,
                     int64_t nkb, int64_t m_pad, ColStat* __restrict__ colstat,
                     const uint8_t* __restrict__ block_mask, int tile_cols, const int32_t* __restrict__ perm,
                     int64_t col_base, int64_t col_end) {
    using D = DirectShape<FP4>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int j = lane % D::WPK;
    const int64_t c = col_base + (int64_t)blockIdx.x * D::COLS + warp * D::COLS_PER_WARP + lane / D::WPK;
    // no early return: the count reduction below shuffles across the warp
    const bool active = c < col_end && (!block_mask || block_mask[c / tile_cols]);
    const bool real = active && c < m;
    const uint64_t* __restrict__ src = words + (real ? (perm ? (int64_t)__ldg(perm + c) : c) : 0) * nw;
    const int64_t kb_stride = m_pad * 128;
    int8_t* const xc = x + c * 128 + j * (128 / D::WPK);
    const int64_t kb0 = (int64_t)blockIdx.y * kDirectKb;
    const int64_t kb1 = kb0 + kDirectKb < nkb ? kb0 + kDirectKb : nkb;
    uint32_t cnt = 0;
    for (int64_t kb = kb0; kb < kb1; kb += kUnr) {
        uint64_t wv[kUnr];
#pragma unroll
        for (int u = 0; u < kUnr; ++u) {
            const int64_t w = D::WPK * (kb + u) + j;
            wv[u] = (real && kb + u < kb1 && w < nw) ? __ldcs(reinterpret_cast<const unsigned long long*>(src + w))
                                                     : 0ull;
        }
#pragma unroll
        for (int u = 0; u < kUnr; ++u) {
            if (active && kb + u < kb1) {
                cnt += __popcll(wv[u]);
                if (x) {  // x == nullptr: column sums only (the word-operand GEMM expands in its producer)
                    if constexpr (FP4) store_fp4_word(xc + (kb + u) * kb_stride, wv[u]);
                    else store_int8_word(xc + (kb + u) * kb_stride, wv[u]);
                }
            }
        }
    }
#pragma unroll
    for (int o = 1; o < D::WPK; o <<= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (j == 0 && real && cnt) atomicAdd(&colstat[c].vi, (int)cnt);
}

// Column sums only (the word-operand path: its GEMM expands the words itself,
// so kernel 1 just counts).  Each warp owns a contiguous chunk of one
// column's words -- kColsumChunk words, 8 loads of 8 bytes in flight per lane,
// 256 contiguous bytes per warp load -- and adds its popcount to the column's
// counter: a streaming read of the words at full DRAM efficiency.
constexpr int kColsumChunk = 2048;
__global__ void __launch_bounds__(256) colsum_words_kernel(const uint64_t* __restrict__ words, int64_t m,
                                                           int64_t nw, int64_t c_begin, int64_t c_end,
                                                           ColStat* __restrict__ colstat) {
    const int lane = threadIdx.x & 31;
    const int64_t chunks = (nw + kColsumChunk - 1) / kColsumChunk;
    const int64_t cols = (c_end < m ? c_end : m) - c_begin;
    const int64_t units = cols * chunks;
    for (int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; u < units;
         u += (int64_t)gridDim.x * blockDim.x / 32) {
        const int64_t c = c_begin + u / chunks;
        const int64_t w0 = (u % chunks) * kColsumChunk;
        const int64_t w1 = w0 + kColsumChunk < nw ? w0 + kColsumChunk : nw;
        const unsigned long long* src = reinterpret_cast<const unsigned long long*>(words + c * nw);
        uint32_t cnt = 0;
        for (int64_t w = w0 + lane; w < w1; w += 32 * 8) {
            unsigned long long v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = w + 32 * k < w1 ? __ldcs(src + w + 32 * k) : 0ull;
#pragma unroll
            for (int k = 0; k < 8; ++k) cnt += __popcll(v[k]);
        }
        cnt = __reduce_add_sync(0xffffffffu, cnt);
        if (lane == 0 && cnt) atomicAdd(&colstat[c].vi, (int)cnt);
    }
}

// Epilogue of kernel 1: per-column statistics from the finished counts.
__global__ void __launch_bounds__(256) colstat_kernel(int64_t n_rows, int64_t m, int64_t c_begin, int64_t c_end,
                                                      int32_t* __restrict__ colsum, ColStat* __restrict__ colstat,
                                                      int fix_s, int2* __restrict__ blkrange) {
    for (int64_t c = c_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < c_end;
         c += (int64_t)gridDim.x * blockDim.x)
        write_colstat(c, (uint32_t)colstat[c].vi, n_rows, c < m, fix_s, colsum, colstat, blkrange);
}

cudaError_t launch_unpack_prep(int64_t n_rows, int64_t m_pad, ColStat* colstat, long long* xlogx, int2* blkrange,
                               float* fixr, int num_sms, cudaStream_t stream, bool table) {
    const int fix_s = xlogx_scale(n_rows);
    const bool have = xlogx != nullptr;  // exact mode has a table: block ranges and mantissa tables too
    int64_t work = (have && table) ? n_rows + 1 : 0;
    if (work < m_pad) work = m_pad;
    int64_t tb = (work + 255) / 256;
    if (tb > (int64_t)num_sms * 16) tb = (int64_t)num_sms * 16;
    unpack_prep_kernel<<<(unsigned)tb, 256, 0, stream>>>(colstat, m_pad, table ? xlogx : nullptr, n_rows, fix_s,
                                                         blkrange, (have && blkrange) ? (int)(m_pad / 128) : 0,
                                                         have ? fixr : nullptr);
    return cudaGetLastError();
}

cudaError_t launch_unpack_range(const uint64_t* words, int64_t n_rows, int64_t m, int64_t nw, int8_t* x, int64_t ld,
                                int64_t m_pad, int32_t* colsum, ColStat* colstat, int2* blkrange, bool fp4,
                                const uint8_t* block_mask, int tile, int64_t c_begin, int64_t c_end, int num_sms,
                                cudaStream_t stream, const int32_t* perm) {
    if (c_begin % kUnpackCols || c_end % kUnpackCols || c_end > m_pad || c_begin >= c_end) return cudaErrorInvalidValue;
    const int fix_s = xlogx_scale(n_rows);
    if (!x) {  // statistics only: a streaming popcount of the columns' words
        const int64_t chunks = (nw + kColsumChunk - 1) / kColsumChunk;
        const int64_t cols = (c_end < m ? c_end : m) - c_begin;
        int64_t blocks = (cols * chunks + 7) / 8;
        if (blocks > (int64_t)num_sms * 16) blocks = (int64_t)num_sms * 16;
        if (blocks > 0)
            colsum_words_kernel<<<(unsigned)blocks, 256, 0, stream>>>(words, m, nw, c_begin, c_end, colstat);
    } else {
        // tools/unpack_bench.py sweeps (r01h, r01m): 32 k-blocks per block and 16
        // loads in flight per thread were best across configs 3-5 (the kernel
        // is memory-latency bound at 50% occupancy: ncu long-scoreboard stalls)
        constexpr int KB = 32, UNR = 16;
        const int64_t nkb = ld / 128;
        const int cols = fp4 ? DirectShape<true>::COLS : DirectShape<false>::COLS;
        const dim3 g2((unsigned)((c_end - c_begin + cols - 1) / cols), (unsigned)((nkb + KB - 1) / KB));
        if (g2.y > 65535) return cudaErrorInvalidValue;
        if (fp4)
            unpack_direct_kernel<true, KB, UNR><<<g2, 256, 0, stream>>>(words, m, nw, x, nkb, m_pad, colstat,
                                                                        block_mask, tile, perm, c_begin, c_end);
        else
            unpack_direct_kernel<false, KB, UNR><<<g2, 256, 0, stream>>>(words, m, nw, x, nkb, m_pad, colstat,
                                                                         block_mask, tile, perm, c_begin, c_end);
    }
    int64_t cb = (c_end - c_begin + 255) / 256;
    if (cb > (int64_t)num_sms * 8) cb = (int64_t)num_sms * 8;
    colstat_kernel<<<(unsigned)cb, 256, 0, stream>>>(n_rows, m, c_begin, c_end, colsum, colstat, fix_s, blkrange);
    return cudaGetLastError();
}

cudaError_t launch_unpack_colsum(const uint64_t* words, int64_t n_rows, int64_t m, int64_t nw, int8_t* x,
                                 int64_t ld, int64_t m_pad, int32_t* colsum, ColStat* colstat, long long* xlogx,
                                 int2* blkrange, float* fixr, bool fp4, const uint8_t* block_mask, int tile,
                                 int num_sms,
                                 cudaStream_t stream, const int32_t* perm) {
    cudaError_t e = launch_unpack_prep(n_rows, m_pad, colstat, xlogx, blkrange, fixr, num_sms, stream);
    if (e != cudaSuccess) return e;
    return launch_unpack_range(words, n_rows, m, nw, x, ld, m_pad, colsum, colstat, xlogx ? blkrange : nullptr, fp4,
                               block_mask, tile, 0, m_pad, num_sms, stream, perm);
}

}  // namespace mib200
