// Column order by column sum, and the pass that puts a result computed in that
// order back into column order.
//
// Why: the fused epilogue's FP64-free table path (c log2 c gathered from a
// fixed-point table) is only fast when the counts of a tile's cells stay in a
// narrow range, i.e. when the tile's column sums are clustered (DESIGN.md,
// "Epilogue math").  With per-column densities spread over [0, 1] (configs 2,
// 4, 5) no tile qualifies in the natural column order and every tile runs the
// FP64 epilogue, serialized behind the MMAs.  Placing the columns in operand
// slots by ascending column sum makes nearly every tile qualify (config 4:
// 0% -> 99% of tiles); MI(i, j) depends only on columns i and j, so the
// result is the same matrix with its rows and columns permuted.
//
//   colsum_kernel      v[c] = popcount of column c (binmat.py:175-177), plus
//                      the global (min, max) of v
//   radix sort         (v, c) pairs by v, stable (cub::DeviceRadixSort), so
//                      ties keep column order: perm[s] = column in slot s
//   inverse_kernel     inv[perm[s]] = s
//   unpermute_kernel   out[r][c] = in[inv[r]][inv[c]]: one CTA per output row
//                      stages the source row in shared memory (coalesced
//                      16-byte loads), then writes the output row in column
//                      order (coalesced stores, gathers from shared memory).
//                      HBM-bound: m^2 esz read + m^2 esz written.
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "mi_kernels.h"

namespace mib200 {

// one warp per column: the column's nw words are one contiguous stream
__global__ void __launch_bounds__(256) colsum_kernel(const uint64_t* __restrict__ words, int64_t m, int64_t nw,
                                                     uint32_t* __restrict__ v, int32_t* __restrict__ idx,
                                                     int* __restrict__ spread) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < m; c += warps) {
        const uint64_t* __restrict__ col = words + c * nw;
        unsigned cnt = 0;
        for (int64_t w = lane; w < nw; w += 32) cnt += __popcll(__ldg(col + w));
#pragma unroll
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (lane == 0) {
            v[c] = cnt;
            idx[c] = (int32_t)c;
            atomicMin(&spread[0], (int)cnt);
            atomicMax(&spread[1], (int)cnt);
        }
    }
}

__global__ void spread_init_kernel(int* spread) {
    spread[0] = 0x7FFFFFFF;
    spread[1] = -1;
}

__global__ void __launch_bounds__(256) inverse_kernel(const int32_t* __restrict__ perm, int32_t* __restrict__ inv,
                                                      int64_t m) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < m; s += (int64_t)gridDim.x * blockDim.x)
        inv[perm[s]] = (int32_t)s;
}

cudaError_t launch_column_order(const uint64_t* words, int64_t n_rows, int64_t m, int32_t* perm, int32_t* inv,
                                int* spread, int num_sms, cudaStream_t stream) {
    const int64_t nw = (n_rows + 63) / 64;
    uint32_t *keys = nullptr, *keys_out = nullptr;
    int32_t* idx = nullptr;
    int* spr = spread;
    void* temp = nullptr;
    size_t temp_bytes = 0;
    int end_bit = 1;
    while (end_bit < 32 && (int64_t(1) << end_bit) <= n_rows) ++end_bit;  // v <= n_rows
    cudaError_t e;
    if ((e = cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, keys, keys_out, idx, perm, (int)m, 0, end_bit,
                                             stream)) != cudaSuccess)
        return e;
    const size_t mb = ((size_t)m * 4 + 255) / 256 * 256;
    {
        // keep the stream-ordered pool's memory cached between calls: with the
        // default release threshold (0) every synchronize hands it back to the
        // driver and the next call pays a fresh mapping (seen: 0.4 -> 4.6 ms)
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = 256ull << 20;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    char* buf = nullptr;
    if ((e = cudaMallocAsync((void**)&buf, 3 * mb + 256 + temp_bytes, stream)) != cudaSuccess) return e;
    keys = reinterpret_cast<uint32_t*>(buf);
    keys_out = reinterpret_cast<uint32_t*>(buf + mb);
    idx = reinterpret_cast<int32_t*>(buf + 2 * mb);
    if (!spr) spr = reinterpret_cast<int*>(buf + 3 * mb);
    temp = buf + 3 * mb + 256;
    spread_init_kernel<<<1, 1, 0, stream>>>(spr);
    int64_t blocks = (m * 32 + 255) / 256;
    if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
    colsum_kernel<<<(unsigned)blocks, 256, 0, stream>>>(words, m, nw, keys, idx, spr);
    e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys, keys_out, idx, perm, (int)m, 0, end_bit, stream);
    if (e == cudaSuccess) {
        int64_t ib = (m + 255) / 256;
        if (ib > (int64_t)num_sms * 8) ib = (int64_t)num_sms * 8;
        inverse_kernel<<<(unsigned)ib, 256, 0, stream>>>(perm, inv, m);
        e = cudaGetLastError();
    }
    cudaError_t e2 = cudaFreeAsync(buf, stream);
    return e != cudaSuccess ? e : e2;
}

// 16 bytes of output gathered from the staged row (register-only: no arrays
// indexed through pointers, which would go to local memory)
template <typename T> struct VecOps;
template <> struct VecOps<unsigned int> {
    using Idx = int4;
    static __device__ __forceinline__ int4 gather(const unsigned int* st, int4 ix) {
        return make_int4((int)st[ix.x], (int)st[ix.y], (int)st[ix.z], (int)st[ix.w]);
    }
};
template <> struct VecOps<unsigned long long> {
    using Idx = int2;
    static __device__ __forceinline__ int4 gather(const unsigned long long* st, int2 ix) {
        const unsigned long long a = st[ix.x], b = st[ix.y];
        return make_int4((int)(unsigned)a, (int)(unsigned)(a >> 32), (int)(unsigned)b, (int)(unsigned)(b >> 32));
    }
};

// out[r][c] = in[inv[r]][inv[c]], r, c < m.  The source row is staged in
// shared memory in chunks of `chunk` elements (one chunk when a whole row
// fits: every shape up to 227 KB per row); with several chunks each pass
// writes the output columns whose source falls in the chunk.
template <typename T>
__global__ void __launch_bounds__(512) unpermute_kernel(const T* __restrict__ in, int64_t ld_in,
                                                         T* __restrict__ out, int64_t ld_out, int m,
                                                         const int32_t* __restrict__ inv, int chunk) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* stage = reinterpret_cast<T*>(smem_raw);
    constexpr int V = 16 / sizeof(T);  // elements per 16-byte vector
    const int tid = threadIdx.x, nthr = blockDim.x;
    const bool vec_out = ((ld_out * (int64_t)sizeof(T)) % 16 == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0) &&
                         ((reinterpret_cast<uintptr_t>(inv) & 15) == 0);
    for (int r = blockIdx.x; r < m; r += gridDim.x) {
        const T* __restrict__ src = in + (int64_t)__ldg(inv + r) * ld_in;
        T* __restrict__ dst = out + (int64_t)r * ld_out;
        for (int s0 = 0; s0 < m; s0 += chunk) {
            const int n = min(chunk, m - s0);
            __syncthreads();  // the previous pass's gathers are done with `stage`
            // stage src[s0, s0 + n): scalar head up to 16-byte alignment, vectors, scalar tail
            const T* s = src + s0;
            int head = (int)(((16 - (reinterpret_cast<uintptr_t>(s) & 15)) & 15) / sizeof(T));
            if ((reinterpret_cast<uintptr_t>(s) % sizeof(T)) != 0) head = n;  // (never for T-aligned rows)
            if (head > n) head = n;
            for (int k = tid; k < head; k += nthr) stage[k] = s[k];
            const int nv = (n - head) / V;
            // stage + head is 16-byte aligned only if head * sizeof(T) is; otherwise copy scalars
            if (((head * sizeof(T)) & 15) == 0) {
                const int4* __restrict__ sv = reinterpret_cast<const int4*>(s + head);
                int4* dv = reinterpret_cast<int4*>(stage + head);
                // 16 independent 16-byte loads in flight per thread before their
                // shared-memory stores (a load -> store -> load chain would
                // leave one load in flight and starve HBM)
                constexpr int U = 16;
                for (int k0 = tid; k0 < nv; k0 += U * nthr) {
                    int4 r[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int k = k0 + u * nthr;
                        if (k < nv) r[u] = __ldcs(sv + k);
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int k = k0 + u * nthr;
                        if (k < nv) dv[k] = r[u];
                    }
                }
            } else {
                for (int k = tid; k < nv * V; k += nthr) stage[head + k] = s[head + k];
            }
            for (int k = head + nv * V + tid; k < n; k += nthr) stage[k] = s[k];
            __syncthreads();
            if (vec_out && n == m) {
                // whole row staged: every output vector is written, B per thread
                // per batch with their index loads issued together
                const int mv = m / V;
                constexpr int B = 8;
                using IV = typename VecOps<T>::Idx;
                for (int q0 = tid; q0 < mv; q0 += B * nthr) {
                    IV iv[B];
#pragma unroll
                    for (int b = 0; b < B; ++b) {
                        const int q = q0 + b * nthr;
                        if (q < mv) iv[b] = __ldg(reinterpret_cast<const IV*>(inv) + q);
                    }
#pragma unroll
                    for (int b = 0; b < B; ++b) {
                        const int q = q0 + b * nthr;
                        if (q < mv) __stcs(reinterpret_cast<int4*>(dst + q * V), VecOps<T>::gather(stage, iv[b]));
                    }
                }
                for (int c = mv * V + tid; c < m; c += nthr) dst[c] = stage[__ldg(inv + c)];
            } else if (vec_out) {
                const int mv = m / V;
                for (int q = tid; q < mv; q += nthr) {
                    alignas(16) T val[V];
                    bool any = false;
#pragma unroll
                    for (int u = 0; u < V; ++u) {
                        const int sidx = __ldg(inv + q * V + u) - s0;
                        const bool in_chunk = (unsigned)sidx < (unsigned)n;
                        val[u] = in_chunk ? stage[sidx] : T(0);
                        any |= in_chunk;
                    }
                    if (n == m) {
                        __stcs(reinterpret_cast<int4*>(dst + q * V), *reinterpret_cast<const int4*>(val));
                    } else if (any) {
#pragma unroll
                        for (int u = 0; u < V; ++u) {
                            const int sidx = __ldg(inv + q * V + u) - s0;
                            if ((unsigned)sidx < (unsigned)n) dst[q * V + u] = val[u];
                        }
                    }
                }
                for (int c = mv * V + tid; c < m; c += nthr) {
                    const int sidx = __ldg(inv + c) - s0;
                    if ((unsigned)sidx < (unsigned)n) dst[c] = stage[sidx];
                }
            } else {
                for (int c = tid; c < m; c += nthr) {
                    const int sidx = __ldg(inv + c) - s0;
                    if ((unsigned)sidx < (unsigned)n) dst[c] = stage[sidx];
                }
            }
        }
    }
}

cudaError_t launch_unpermute(const void* in, int64_t ld_in, void* out, int64_t ld_out, int64_t m, int esz,
                             const int32_t* inv, int num_sms, int smem_bytes, int ctas_per_sm, cudaStream_t stream) {
    const int max_elems = smem_bytes / esz;
    const int chunk = (int)(m < max_elems ? m : max_elems);
    const size_t shm = (size_t)chunk * esz;
    int64_t grid = (int64_t)num_sms * ctas_per_sm;
    if (grid > m) grid = m;
    const int threads = std::max(128, 512 / ctas_per_sm / 32 * 32);
    cudaError_t e;
    if (esz == 8) {
        if ((e = cudaFuncSetAttribute(unpermute_kernel<unsigned long long>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)shm)) != cudaSuccess)
            return e;
        unpermute_kernel<unsigned long long><<<(unsigned)grid, threads, shm, stream>>>(
            static_cast<const unsigned long long*>(in), ld_in, static_cast<unsigned long long*>(out), ld_out, (int)m, inv, chunk);
    } else {
        if ((e = cudaFuncSetAttribute(unpermute_kernel<unsigned int>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)shm)) != cudaSuccess)
            return e;
        unpermute_kernel<unsigned int><<<(unsigned)grid, threads, shm, stream>>>(
            static_cast<const unsigned int*>(in), ld_in, static_cast<unsigned int*>(out), ld_out, (int)m, inv, chunk);
    }
    return cudaGetLastError();
}

}  // namespace mib200
