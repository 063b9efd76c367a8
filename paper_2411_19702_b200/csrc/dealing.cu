// Tile dealing: the upper-triangle tile order and each rank's share
// (host-side logic behind mi_tile_list / mi_rank_blocks; no device work).
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

namespace mib200 {
namespace capi {

// Tile rows/columns that contain real columns (the operand is padded to 256).
int64_t tiles_per_side(int64_t n_cols) {
    const int64_t t = mi_tile_size();
    return (n_cols + t - 1) / t;
}

// Banded upper-triangle order: within a band of `band` tile rows, sweep J and
// then the band's rows, so tiles that run concurrently share operand blocks.
// `first` > 0 makes the first band that many rows (1 for the host path: tile
// row 0 completes in the first wave, so the D2H of finished rows starts early).
std::vector<int32_t> all_tiles(int64_t T, int band, int first) {
    std::vector<int32_t> v;
    v.reserve((size_t)(T * (T + 1)));
    for (int64_t I0 = 0; I0 < T;) {
        const int64_t b = (I0 == 0 && first > 0) ? first : band;
        for (int64_t J = I0; J < T; ++J)
            for (int64_t I = I0; I < I0 + b && I <= J; ++I) {
                v.push_back((int32_t)I);
                v.push_back((int32_t)J);
            }
        I0 += b;
    }
    return v;
}

// A rank's tiles.  Round robin over the banded order (every rank touches
// nearly every column block), except for 4 ranks (below: each rank holds 3 of
// 4 column groups) and 8 ranks ("shard" knob, T >= 8): the
// column blocks form 4 groups; ranks 0-5 take the 6 off-diagonal group pairs
// (g, h), ranks 6 and 7 two diagonal groups each ((0,0)+(3,3), (1,1)+(2,2)).
// Every rank then reads -- and unpacks -- only 2 of the 4 groups (half of X),
// at a load imbalance of ~4/T (off-diagonal s^2 tiles vs s^2 + s).
std::vector<int32_t> rank_tiles(int64_t T, int rank, int world, int band) {
    const std::vector<int32_t> all = all_tiles(T, band);
    const int64_t total = (int64_t)all.size() / 2;
    std::vector<int32_t> v;
    if (world == 8 && T >= 8 && tuning().shard) {
        auto group = [&](int64_t b) { return (int)((b * 4) / T); };
        static const int pairs[8][4] = {{0, 1, -1, -1}, {0, 2, -1, -1}, {0, 3, -1, -1}, {1, 2, -1, -1},
                                        {1, 3, -1, -1}, {2, 3, -1, -1}, {0, 0, 3, 3}, {1, 1, 2, 2}};
        std::vector<std::vector<int32_t>> share(8);
        for (int64_t k = 0; k < total; ++k) {
            const int gi = group(all[2 * k]), gj = group(all[2 * k + 1]);
            for (int r = 0; r < 8; ++r) {
                const int* pr = pairs[r];
                if ((gi == pr[0] && gj == pr[1]) || (pr[2] >= 0 && gi == pr[2] && gj == pr[3])) {
                    share[r].push_back(all[2 * k]);
                    share[r].push_back(all[2 * k + 1]);
                    break;
                }
            }
        }
        // The two diagonal-group ranks hold s(s + 1) tiles against s^2: hand
        // their surplus (from the end of their lists) to off-diagonal ranks
        // that already hold that group's blocks -- no extra unpack -- always
        // to the least loaded one, until no rank exceeds ceil(total / 8).
        const size_t cap = (size_t)((total + 7) / 8);
        auto holds = [&](int r, int g) { return pairs[r][0] == g || pairs[r][1] == g; };
        for (int d = 6; d < 8; ++d) {
            while (share[d].size() / 2 > cap) {
                int best_r = -1;
                int64_t best_k = -1;
                for (int gsel = 0; gsel < 2; ++gsel) {
                    const int g = pairs[d][2 * gsel];
                    int r_min = -1;
                    for (int r = 0; r < 6; ++r)
                        if (holds(r, g) && (r_min < 0 || share[r].size() < share[r_min].size())) r_min = r;
                    if (r_min < 0 || share[r_min].size() / 2 >= cap) continue;
                    if (best_r >= 0 && share[best_r].size() <= share[r_min].size()) continue;
                    for (int64_t k = (int64_t)share[d].size() / 2 - 1; k >= 0; --k)
                        if (group(share[d][2 * k]) == g) {
                            best_r = r_min;
                            best_k = k;
                            break;
                        }
                }
                if (best_r < 0) break;
                share[best_r].push_back(share[d][2 * best_k]);
                share[best_r].push_back(share[d][2 * best_k + 1]);
                share[d].erase(share[d].begin() + 2 * best_k, share[d].begin() + 2 * best_k + 2);
            }
        }
        return share[rank];
    }
    if (world == 4 && T >= 16 && tuning().shard) {
        // 4 column groups; rank r holds every group but r (3/4 of X).  Every
        // group pair (g, h) lies in the two or three ranks that hold both;
        // tiles go, in the banded order, to the least-loaded of those, so the
        // shares differ by at most a tile or two and each rank unpacks 3/4 of X
        // instead of all of it.
        auto group = [&](int64_t b) { return (int)((b * 4) / T); };
        // each group pair's tiles go round robin over the ranks that hold
        // both groups (2 for an off-diagonal pair, 3 for a diagonal one), so
        // every rank gets half of three off-diagonal pairs and a third of three
        // diagonal ones; the rank's list keeps the banded order
        std::vector<int8_t> owner((size_t)total, -1);
        int cnt[4][4] = {};
        for (int64_t k = 0; k < total; ++k) {
            const int gi = group(all[2 * k]), gj = group(all[2 * k + 1]);
            int elig[3], ne = 0;
            for (int r = 0; r < 4; ++r)
                if (r != gi && r != gj) elig[ne++] = r;
            owner[(size_t)k] = (int8_t)elig[cnt[gi][gj]++ % ne];
        }
        // unequal group sizes (T % 4 != 0) leave a small imbalance: move tiles,
        // from the end of the order, off the most loaded rank to the least
        // loaded rank that also holds both of their groups
        int64_t load[4] = {0, 0, 0, 0};
        for (int64_t k = 0; k < total; ++k) ++load[owner[(size_t)k]];
        for (int64_t moves = 0; moves < total; ++moves) {
            int hi = 0;
            for (int r = 1; r < 4; ++r)
                if (load[r] > load[hi]) hi = r;
            bool moved = false;
            for (int64_t k = total - 1; k >= 0 && !moved; --k) {
                if (owner[(size_t)k] != hi) continue;
                const int gi = group(all[2 * k]), gj = group(all[2 * k + 1]);
                int lo = -1;
                for (int r = 0; r < 4; ++r)
                    if (r != gi && r != gj && r != hi && load[r] + 1 < load[hi] && (lo < 0 || load[r] < load[lo]))
                        lo = r;
                if (lo < 0) continue;
                owner[(size_t)k] = (int8_t)lo;
                --load[hi];
                ++load[lo];
                moved = true;
            }
            if (!moved) break;
        }
        for (int64_t k = 0; k < total; ++k)
            if (owner[(size_t)k] == rank) {
                v.push_back(all[2 * k]);
                v.push_back(all[2 * k + 1]);
            }
        return v;
    }
    for (int64_t g = rank; g < total; g += world) {
        v.push_back(all[2 * g]);
        v.push_back(all[2 * g + 1]);
    }
    return v;
}

}  // namespace capi
}  // namespace mib200

extern "C" {

int64_t mi_num_tiles(int64_t n_cols) {
    const int64_t T = tiles_per_side(n_cols);
    return T * (T + 1) / 2;
}

int64_t mi_tile_list(int64_t n_cols, int rank, int world, int band, int32_t* tiles_out, int64_t capacity) {
    if (n_cols < 1) return -fail(MI_ERR_DIMENSION, "n_cols must be >= 1");
    if (world < 1 || rank < 0 || rank >= world)
        return -fail(MI_ERR_DOMAIN, "bad rank %d of world %d", rank, world);
    if (band <= 0) band = tile_band();
    const int64_t T = tiles_per_side(n_cols);
    const std::vector<int32_t> mine = rank_tiles(T, rank, world, band);
    const int64_t count = (int64_t)mine.size() / 2;
    if (tiles_out) {
        if (count > capacity) return -fail(MI_ERR_DIMENSION, "tile buffer too small");
        memcpy(tiles_out, mine.data(), mine.size() * sizeof(int32_t));
    }
    return count;
}

int64_t mi_rank_blocks(int64_t n_cols, int rank, int world, uint8_t* mask_out, int64_t capacity) {
    if (n_cols < 1) return -fail(MI_ERR_DIMENSION, "n_cols must be >= 1");
    if (world < 1 || rank < 0 || rank >= world)
        return -fail(MI_ERR_DOMAIN, "bad rank %d of world %d", rank, world);
    const int64_t T = tiles_per_side(n_cols);
    if (!mask_out) return T;
    if (capacity < T) return -fail(MI_ERR_DIMENSION, "mask buffer too small");
    memset(mask_out, 0, (size_t)T);
    const std::vector<int32_t> mine = rank_tiles(T, rank, world, tile_band());
    for (size_t k = 0; k < mine.size(); ++k) mask_out[mine[k]] = 1;
    int64_t used = 0;
    for (int64_t b = 0; b < T; ++b) used += mask_out[b];
    return used;
}

}  // extern "C"
