// Synthetic input generator, writing the packed-word layout directly.
//
// Bit-exact with the reference's datagen.generate (datagen.py:44-73):
// cell (r, c) consumes draw k = r * m + c + 1 of the splitmix64 stream whose
// state for draw k is seed + k * 0x9E3779B97F4A7C15, and is 1 iff the draw is
// below ceil(p_c * 2^64).  Per-column kinds add the BASELINE config recipes
// (SURVEY 8(d)): constant columns and noisy copies (target = source XOR a
// Bernoulli flip drawn from the stream seeded with seed ^ 0xA5A5...A5 at the
// target's own cell index).
//
// One thread per output word (64 rows of one column), coalesced along the
// column's word stream; no (N x m) byte matrix is ever materialised.
#include <cuda_runtime.h>
#include <cstdint>

#include "mi_kernels.h"

namespace mib200 {

__device__ __forceinline__ uint64_t splitmix64_draw(uint64_t seed, uint64_t k) {
    uint64_t z = seed + k * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// kind: 0 Bernoulli(thr), 1 all zero, 2 all one, 3 copy of src column with flips
__global__ void generate_words_kernel(uint64_t* __restrict__ words, int64_t n_rows, int64_t m, int64_t nw,
                                      uint64_t seed, const uint64_t* __restrict__ thr,
                                      const uint8_t* __restrict__ kind, const int32_t* __restrict__ src,
                                      uint64_t flip_thr, uint64_t flip_seed) {
    const int64_t total = m * nw;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = idx / nw;
        const int64_t w = idx - c * nw;
        const int64_t r0 = w * 64;
        int64_t nr = n_rows - r0;
        if (nr > 64) nr = 64;
        const uint8_t kd = kind[c];
        uint64_t out = 0;
        if (kd == 2) {
            out = (nr == 64) ? ~0ull : ((1ull << nr) - 1ull);
        } else if (kd == 0) {
            const uint64_t t = thr[c];
            for (int b = 0; b < nr; ++b) {
                const uint64_t k = (uint64_t)(r0 + b) * (uint64_t)m + (uint64_t)c + 1ull;
                out |= (uint64_t)(splitmix64_draw(seed, k) < t) << b;
            }
        } else if (kd == 3) {
            const int64_t s = src[c];
            const uint64_t t = thr[s];
            for (int b = 0; b < nr; ++b) {
                const uint64_t row = (uint64_t)(r0 + b) * (uint64_t)m;
                const uint64_t sb = splitmix64_draw(seed, row + (uint64_t)s + 1ull) < t;
                const uint64_t fb = splitmix64_draw(flip_seed, row + (uint64_t)c + 1ull) < flip_thr;
                out |= (sb ^ fb) << b;
            }
        }
        words[idx] = out;
    }
}

cudaError_t launch_generate_words(uint64_t* words, int64_t n_rows, int64_t m, uint64_t seed,
                                  const uint64_t* col_threshold, const uint8_t* col_kind,
                                  const int32_t* col_src, uint64_t flip_threshold, uint64_t flip_seed,
                                  cudaStream_t stream) {
    const int64_t nw = (n_rows + 63) / 64;
    const int64_t total = m * nw;
    const int threads = 256;
    int64_t blocks = (total + threads - 1) / threads;
    if (blocks > 148 * 64) blocks = 148 * 64;
    if (blocks < 1) blocks = 1;
    generate_words_kernel<<<(unsigned)blocks, threads, 0, stream>>>(
        words, n_rows, m, nw, seed, col_threshold, col_kind, col_src, flip_threshold, flip_seed);
    return cudaGetLastError();
}

}  // namespace mib200
