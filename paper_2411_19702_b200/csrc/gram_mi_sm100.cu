// Kernel 2+3: symmetric upper-triangle int8 Gram on tcgen05 with the mutual-
// information epilogue fused onto the TMEM accumulators.
//
// Replaces, for one output tile at a time, the reference's
//   _kernels.gram_ones_kernel        _kernels.py:48-61   (G11 = D^T D by AND+popcount)
//   gram.gram_complete_optimized     gram.py:88-111      (g00 / g01 in closed form)
//   engine.probabilities             engine.py:93-102
//   engine.mi_from_probabilities     engine.py:116-141   (four cells, fixed order, mirror)
// so that G never reaches HBM: each (I <= J) tile of G lives in TMEM, is read
// once by the epilogue warps and written out as MI(I,J) and its mirror
// MI(J,I).
//
// Layout: X is the K-major int8 expansion of the bit-packed
// columns, X[c][r] = bit r of column c, shape m_pad x N_pad (N_pad % 128 == 0,
// m_pad % 256 == 0, zero padded).  Both GEMM operands are row blocks of X.
//
// Warp roles (384 threads, one CTA per SM, persistent over a static tile list):
//   warp 0      TMA producer (one lane): A = X[rows of I], B = X[rows of J]
//   warp 1      MMA issuer (one lane, leader CTA only when CG == 2)
//   warp 2      TMEM allocator
//   warp 3      idle
//   warps 4-11  epilogue: tcgen05.ld -> counts -> fp64 MI -> global
// CG == 2: a CTA pair (cluster of 2) computes a 256x256 tile with
// tcgen05.mma.cta_group::2 (M=256, N=256); each CTA stages half of A and half
// of B, and owns 128 accumulator rows.  CG == 1: 128x128 tiles on one SM.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "ptx.cuh"
#include "mi_kernels.h"

namespace mib200 {

constexpr int kThreads = 384;
constexpr int kEpiWarp0 = 4;
constexpr int kNumEpiWarps = 8;
constexpr int kBK = 128;                 // K bytes per pipeline stage (= 128B swizzle span)
constexpr int kStageHalfBytes = 128 * kBK;  // one 128-row operand half: 16 KB
constexpr int kStages = 6;

template <int CG>
struct Cfg {
    static constexpr int TS = 128 * CG;           // square output tile
    static constexpr int MMA_M = 128 * CG;
    static constexpr int MMA_N = 128 * CG;
    static constexpr int ACC_COLS = MMA_N;        // TMEM columns per accumulator
    static constexpr int TMEM_COLS = 2 * ACC_COLS;  // double-buffered
    static constexpr int HALF_COLS = ACC_COLS / 2;  // columns per epilogue warp
    static constexpr int CHUNKS = HALF_COLS / 32;
    static constexpr uint32_t STAGE_TX = CG * 2 * kStageHalfBytes;  // bytes landing per stage
};

struct SmemLayout {
    static constexpr uint32_t a_off = 0;
    static constexpr uint32_t b_off = kStages * kStageHalfBytes;
    static constexpr uint32_t bar_off = 2 * kStages * kStageHalfBytes;
    // full[kStages], empty[kStages], tfull[2], tempty[2], tmem slot
    static constexpr uint32_t bytes = bar_off + (2 * kStages + 4) * 8 + 16;
};
constexpr uint32_t kSmemBytes = SmemLayout::bytes + 1024;  // + alignment slack

// ---------------------------------------------------------------- epilogue math

// c * log2(c * N / (a * b)) with 0 * log 0 = 0.  c, a, b, N are exact
// integers in fp64 (all < 2^31, products < 2^53 for N < 9.4e7), so the ratio
// is one correctly rounded division.  Summing these over the four cells and
// dividing by N gives sum_cells p * log2(p / (p_a p_b)) (engine.py:105-109,
// 131-136); e.g. an identical balanced pair yields exactly 1.0 and an
// independent one exactly 0.0, like the reference.
__device__ __forceinline__ double xlog2r(double c, double ab, double dN) {
    return c > 0.0 ? c * log2((c * dN) / ab) : 0.0;
}

// MI of one pair in orientation (i, j): vi = ones in column i (row of the
// tile), vj = ones in column j.  Cells in the reference's fixed order
// (1,1), (1,0), (0,1), (0,0) (engine.py:124-129).
template <int MODE>
__device__ __forceinline__ double mi_pair(int g, int vi, int vj, double dN, int N, double eps) {
    const double c11 = (double)g;
    const double c10 = (double)(vi - g);
    const double c01 = (double)(vj - g);
    const double c00 = (double)(N - vi - vj + g);
    const double a1 = (double)vi, a0 = (double)(N - vi);
    const double b1 = (double)vj, b0 = (double)(N - vj);
    if constexpr (MODE == MI_MODE_EXACT) {
        double s = xlog2r(c11, a1 * b1, dN);
        s += xlog2r(c10, a1 * b0, dN);
        s += xlog2r(c01, a0 * b1, dN);
        s += xlog2r(c00, a0 * b0, dN);
        return s / dN;
    } else {
        // engine.py:112-113: p * log2((p + eps) / (e + eps)), p = count / n,
        // e = (a / n) * (b / n) -- evaluated with the reference's operations.
        const double pa1 = a1 / dN, pa0 = a0 / dN, pb1 = b1 / dN, pb0 = b0 / dN;
        double p, s;
        p = c11 / dN; s = p * log2((p + eps) / (pa1 * pb1 + eps));
        p = c10 / dN; s += p * log2((p + eps) / (pa1 * pb0 + eps));
        p = c01 / dN; s += p * log2((p + eps) / (pa0 * pb1 + eps));
        p = c00 / dN; s += p * log2((p + eps) / (pa0 * pb0 + eps));
        return s;
    }
}

template <int OUT>
struct OutT;
template <> struct OutT<MI_OUT_COUNTS> { using T = int32_t; };
template <> struct OutT<MI_OUT_F64> { using T = double; };
template <> struct OutT<MI_OUT_F32> { using T = float; };


// 32 consecutive outputs of one thread as 16-byte vector stores.
__device__ __forceinline__ void store_row32(double* dst, const double (&v)[32]) {
#pragma unroll
    for (int k = 0; k < 32; k += 2) *reinterpret_cast<double2*>(dst + k) = make_double2(v[k], v[k + 1]);
}
__device__ __forceinline__ void store_row32(float* dst, const float (&v)[32]) {
#pragma unroll
    for (int k = 0; k < 32; k += 4)
        *reinterpret_cast<float4*>(dst + k) = make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]);
}
__device__ __forceinline__ void store_row32(int32_t* dst, const int32_t (&v)[32]) {
#pragma unroll
    for (int k = 0; k < 32; k += 4)
        *reinterpret_cast<int4*>(dst + k) = make_int4(v[k], v[k + 1], v[k + 2], v[k + 3]);
}

// ---------------------------------------------------------------- the kernel

template <int CG, int OUT, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
gram_mi_kernel(const __grid_constant__ CUtensorMap tmap_x, const GramMiParams p) {
    using C = Cfg<CG>;
    using T = typename OutT<OUT>::T;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    const uint32_t base = (raw_addr + 1023u) & ~1023u;  // SW128 needs 1024-B alignment
    uint8_t* const smem = smem_raw + (base - raw_addr);

    const uint32_t sA = base + SmemLayout::a_off;
    const uint32_t sB = base + SmemLayout::b_off;
    const uint32_t bar0 = base + SmemLayout::bar_off;
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto empty_bar = [&](int s) { return bar0 + 8u * (kStages + s); };
    auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * kStages + a); };
    auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * kStages + 2 + a); };
    const uint32_t tmem_slot = bar0 + 8u * (2 * kStages + 4);
    volatile uint32_t* tmem_slot_ptr =
        reinterpret_cast<volatile uint32_t*>(smem + SmemLayout::bar_off + 8 * (2 * kStages + 4));

    const int warp = threadIdx.x / 32;
    const uint32_t lane = lane_id();
    const uint32_t rank = (CG == 2) ? cluster_ctarank() : 0u;
    const int cluster = (CG == 2) ? (int)cluster_id_x() : (int)blockIdx.x;
    const int n_clusters = (CG == 2) ? (int)num_clusters_x() : (int)gridDim.x;

    // ---- one-time setup
    if (threadIdx.x == 0) {
        prefetch_tmap(&tmap_x);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull_bar(a), 1);
            mbar_init(tempty_bar(a), CG * kNumEpiWarps);
        }
        fence_mbarrier_init();
    }
    if (warp == 2) tmem_alloc<CG>(tmem_slot, C::TMEM_COLS);
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot_ptr;

    const int nkb = p.num_k_blocks;

    if (warp == 0) {
        // ================= TMA producer =================
        if (lane == 0) {
            const uint64_t policy = l2_policy_evict_last();
            // CG == 2: both CTAs signal the leader's full barrier.
            const uint32_t fb_rank = (CG == 2) ? 0u : rank;
            int s = 0;
            uint32_t ph = 0;
            for (int t = cluster; t < p.n_tiles; t += n_clusters) {
                const int2 tile = p.tiles[t];
                const int rowA = tile.x * C::TS + (int)rank * 128;
                const int rowB = tile.y * C::TS + (int)rank * 128;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(empty_bar(s), ph ^ 1u);
                    const uint32_t fb = (CG == 2) ? map_to_cta(full_bar(s), fb_rank) : full_bar(s);
                    if (rank == 0) mbar_arrive_expect_tx(full_bar(s), C::STAGE_TX);
                    tma_load_2d<CG>(sA + s * kStageHalfBytes, &tmap_x, fb, kb * kBK, rowA, policy);
                    tma_load_2d<CG>(sB + s * kStageHalfBytes, &tmap_x, fb, kb * kBK, rowB, policy);
                    if (++s == kStages) { s = 0; ph ^= 1u; }
                }
            }
            // drain: the last commit of every stage must land before exit
            for (int i = 0; i < kStages; ++i) {
                mbar_wait(empty_bar(s), ph ^ 1u);
                if (++s == kStages) { s = 0; ph ^= 1u; }
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer =================
        if (rank == 0 && lane == 0) {
            constexpr uint32_t idesc = umma_idesc_i8(C::MMA_M, C::MMA_N);
            int s = 0;
            uint32_t ph = 0;
            int acc = 0;
            uint32_t aph = 0;
            for (int t = cluster; t < p.n_tiles; t += n_clusters) {
                mbar_wait(tempty_bar(acc), aph ^ 1u);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + (uint32_t)(acc * C::ACC_COLS);
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(full_bar(s), ph);
                    tc_fence_after();
                    const uint64_t adesc = umma_desc_sw128_kmajor(sA + s * kStageHalfBytes);
                    const uint64_t bdesc = umma_desc_sw128_kmajor(sB + s * kStageHalfBytes);
#pragma unroll
                    for (int k = 0; k < kBK / 32; ++k) {
                        // advance 32 bytes (one K=32 int8 step) inside the swizzle atom
                        umma_i8<CG>(d_tmem, adesc + 2u * k, bdesc + 2u * k, idesc,
                                    (kb | k) != 0 ? 1u : 0u);
                    }
                    umma_commit<CG>(empty_bar(s));  // frees the smem slot (both CTAs)
                    if (++s == kStages) { s = 0; ph ^= 1u; }
                }
                umma_commit<CG>(tfull_bar(acc));  // accumulator ready (both CTAs)
                if (++acc == 2) { acc = 0; aph ^= 1u; }
            }
        }
    } else if (warp >= kEpiWarp0) {
        // ================= epilogue =================
        const int q = warp & 3;                    // TMEM lane quadrant of this warp
        const int h = (warp - kEpiWarp0) >> 2;     // which half of the accumulator columns
        const int row_local = q * 32 + (int)lane;
        const int m = p.m;
        const int N = p.n_rows;
        const double dN = (double)N;
        const int64_t ld = p.ld_out;
        T* __restrict__ out = reinterpret_cast<T*>(p.out);
        const uint32_t tempty_leader0 = (CG == 2) ? map_to_cta(tempty_bar(0), 0) : tempty_bar(0);
        const uint32_t tempty_leader1 = (CG == 2) ? map_to_cta(tempty_bar(1), 0) : tempty_bar(1);
        int acc = 0;
        uint32_t aph = 0;
        for (int t = cluster; t < p.n_tiles; t += n_clusters) {
            const int2 tile = p.tiles[t];
            const bool diag = tile.x == tile.y;
            const int i = tile.x * C::TS + (int)rank * 128 + row_local;
            const int vi = (i < m) ? __ldg(p.colsum + i) : 0;
            mbar_wait(tfull_bar(acc), aph);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < C::CHUNKS; ++c) {
                const int col0 = h * C::HALF_COLS + c * 32;
                const int j0 = tile.y * C::TS + col0;
                uint32_t r[32];
                tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) +
                                       (uint32_t)(acc * C::ACC_COLS + col0),
                                   r);
                tmem_ld_wait(r);
                T val[32];
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    const int j = j0 + k;
                    const int g = (int)r[k];
                    if constexpr (OUT == MI_OUT_COUNTS) {
                        val[k] = g;
                    } else {
                        const int vj = (j < m) ? __ldg(p.colsum + j) : 0;
                        // compute every element in (min, max) orientation so the
                        // mirrored halves of diagonal tiles are bit-identical
                        const bool swap = diag && (j < i);
                        double x = mi_pair<MODE>(g, swap ? vj : vi, swap ? vi : vj, dN, N, p.eps);
                        if (!p.include_diagonal && i == j) x = 0.0;
                        val[k] = (T)x;
                    }
                }
                if (i < m) {
                    // direct tile: row i, columns j0 .. j0+31
                    T* dst = out + (int64_t)i * ld + j0;
                    if (j0 + 32 <= m && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
                        store_row32(dst, val);
                    } else {
#pragma unroll
                        for (int k = 0; k < 32; ++k)
                            if (j0 + k < m) dst[k] = val[k];
                    }
                    // mirror tile: row j, column i (coalesced across the warp)
                    if (!diag) {
#pragma unroll
                        for (int k = 0; k < 32; ++k)
                            if (j0 + k < m) out[(int64_t)(j0 + k) * ld + i] = val[k];
                    }
                }
            }
            // hand the accumulator back to the MMA warp
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(acc == 0 ? tempty_leader0 : tempty_leader1);
            if (++acc == 2) { acc = 0; aph ^= 1u; }
        }
    }

    // ---- teardown
    __syncwarp();
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc<CG>(tmem_base, C::TMEM_COLS);
}

// ---------------------------------------------------------------- launch

template <int CG, int OUT, int MODE>
static cudaError_t launch_impl(const CUtensorMap& tmap, const GramMiParams& p, int num_sms,
                               cudaStream_t stream) {
    auto kern = gram_mi_kernel<CG, OUT, MODE>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSmemBytes);
    if (e != cudaSuccess) return e;
    const int max_clusters = num_sms / CG;
    int clusters = p.n_tiles < max_clusters ? p.n_tiles : max_clusters;
    if (clusters < 1) clusters = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(clusters * CG, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, tmap, p);
}

cudaError_t launch_gram_mi(int cg, int out_kind, int mode, const CUtensorMap& tmap,
                           const GramMiParams& p, int num_sms, cudaStream_t stream) {
#define MI_DISPATCH(CGV, OV, MV) \
    if (cg == CGV && out_kind == OV && mode == MV) return launch_impl<CGV, OV, MV>(tmap, p, num_sms, stream);
    MI_DISPATCH(2, MI_OUT_F64, MI_MODE_EXACT)
    MI_DISPATCH(2, MI_OUT_F64, MI_MODE_EPSILON)
    MI_DISPATCH(2, MI_OUT_F32, MI_MODE_EXACT)
    MI_DISPATCH(2, MI_OUT_F32, MI_MODE_EPSILON)
    MI_DISPATCH(2, MI_OUT_COUNTS, MI_MODE_EXACT)
    MI_DISPATCH(1, MI_OUT_F64, MI_MODE_EXACT)
    MI_DISPATCH(1, MI_OUT_F64, MI_MODE_EPSILON)
    MI_DISPATCH(1, MI_OUT_F32, MI_MODE_EXACT)
    MI_DISPATCH(1, MI_OUT_F32, MI_MODE_EPSILON)
    MI_DISPATCH(1, MI_OUT_COUNTS, MI_MODE_EXACT)
#undef MI_DISPATCH
    return cudaErrorInvalidValue;
}

int gram_mi_tile_size(int cg) { return 128 * cg; }
uint32_t gram_mi_smem_bytes() { return kSmemBytes; }

}  // namespace mib200
