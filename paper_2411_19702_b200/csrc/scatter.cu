// Gather of the sharded result (mi_scatter_tiles): tile-major shards written
// by the fused kernel (MI_TILE_MAJOR: each rank's tiles, no mirrors) placed
// into a full row-major m x m matrix with their mirrors -- on a device, or
// straight into pinned host memory over PCIe (zero-copy), so every rank of a
// node writes its own share of one host matrix over its own link.
//
// One CTA per 64 x 64 sub-block of a tile: the block is staged in shared
// memory (padded rows: conflict-free transposed reads), written back as
// 64-element row runs at (I, J) and, transposed, at (J, I).  Bandwidth-bound:
// 2 x esz bytes written and esz read per element (HBM or PCIe).
#include <cuda_runtime.h>
#include <cstdint>

#include "mi_kernels.h"

namespace mib200 {

namespace {

constexpr int kSub = 64;

template <typename T>
__global__ void __launch_bounds__(256) scatter_tiles_kernel(const T* __restrict__ src, const int2* __restrict__ tiles,
                                                            int ts, int64_t m, T* __restrict__ dst, int64_t ld,
                                                            int mirror) {
    __shared__ T blk[kSub][kSub + 1];
    const int per_side = ts / kSub;
    const int t = blockIdx.x;
    const int sb = blockIdx.y;  // sub-block of the tile
    const int sr = (sb / per_side) * kSub, sc = (sb % per_side) * kSub;
    const int2 tile = tiles[t];
    const int64_t r0 = (int64_t)tile.x * ts + sr, c0 = (int64_t)tile.y * ts + sc;
    if (r0 >= m || c0 >= m) return;
    const T* s = src + (int64_t)t * ts * ts + (int64_t)sr * ts + sc;
    const int lane = threadIdx.x & 63, row0 = threadIdx.x >> 6;  // 4 rows of 64 per pass
    for (int r = row0; r < kSub; r += 4) blk[r][lane] = s[(int64_t)r * ts + lane];
    __syncthreads();
    // direct block: rows r0 + r, columns c0 + lane
    for (int r = row0; r < kSub; r += 4)
        if (r0 + r < m && c0 + lane < m) dst[(r0 + r) * ld + c0 + lane] = blk[r][lane];
    if (!mirror || tile.x == tile.y) return;
    // mirror block: rows c0 + r, columns r0 + lane = blk[lane][r]
    for (int r = row0; r < kSub; r += 4)
        if (c0 + r < m && r0 + lane < m) dst[(c0 + r) * ld + r0 + lane] = blk[lane][r];
}

}  // namespace

cudaError_t launch_scatter_tiles(const void* src, const int32_t* tiles, int64_t n_tiles, int ts, int64_t m, int esz,
                                 void* dst, int64_t ld, bool mirror, cudaStream_t stream) {
    if (n_tiles == 0) return cudaSuccess;
    const dim3 grid((unsigned)n_tiles, (unsigned)((ts / kSub) * (ts / kSub)));
    const int2* t = reinterpret_cast<const int2*>(tiles);
    if (esz == 8)
        scatter_tiles_kernel<double><<<grid, 256, 0, stream>>>(static_cast<const double*>(src), t, ts, m,
                                                               static_cast<double*>(dst), ld, mirror ? 1 : 0);
    else
        scatter_tiles_kernel<float><<<grid, 256, 0, stream>>>(static_cast<const float*>(src), t, ts, m,
                                                              static_cast<float*>(dst), ld, mirror ? 1 : 0);
    return cudaGetLastError();
}

}  // namespace mib200
