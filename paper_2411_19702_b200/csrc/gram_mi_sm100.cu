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
// columns, X[c][r] = bit r of column c, stored k-blocked as
// [N_pad/128][m_pad][128 bytes] (N_pad % 128 == 0, m_pad % 256 == 0, zero
// padded) so each 128 x 128 TMA box is one contiguous 16 KB chunk.  Both GEMM
// operands are row blocks of X.
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

#include "milog.cuh"
#include "mi_kernels.h"
#include "ptx.cuh"

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
    static constexpr uint32_t tab_off = 2 * kStages * kStageHalfBytes;   // log2 table, 2 KB
    static constexpr uint32_t bar_off = tab_off + 128 * 16;
    // full[kStages], empty[kStages], tfull[2], tempty[2], tmem slot
    static constexpr uint32_t bytes = bar_off + (2 * kStages + 4) * 8 + 16;
};
constexpr uint32_t kSmemBytes = SmemLayout::bytes + 1024;  // + alignment slack

// ---------------------------------------------------------------- epilogue math

// Exact-mode MI of one pair (engine.py:105-109,116-141), from integer counts.
// Each cell contributes c * log2(c N / (a b)), summed in the reference's fixed
// order (1,1), (1,0), (0,1), (0,0) and divided by N at the end.  The log of the
// ratio is assembled as integer exponents plus table-driven mantissa fractions
// (milog.cuh): L = (e_c + e_N - e_a - e_b) + (((f_c + f_N) - f_a) - f_b), with
// the marginal logs precomputed once per column by kernel 1.  Identical
// mantissas cancel exactly, so an identical balanced pair gives exactly 1.0 and
// an independent one (c N == a b with equal mantissas) exactly 0.0, as in the
// reference; elsewhere the result is within ~1e-15 of the reference's value.
struct Marg {
    double f1, f0;  // log2 fractions of a1 = v and a0 = N - v
    int e1, e0;     // and their exponents
    int v;
};

__device__ __forceinline__ Marg load_marg(const ColStat* __restrict__ cs, int idx) {
    const double2 f = __ldg(reinterpret_cast<const double2*>(cs + idx));
    const int4 e = __ldg(reinterpret_cast<const int4*>(cs + idx) + 1);
    return Marg{f.x, f.y, e.x, e.y, e.z};
}

__device__ __forceinline__ double cell_term(int c, int ea, double fa, int eb, double fb, int eN, double fN,
                                            const double2* __restrict__ tab) {
    const double dc = (double)(c > 0 ? c : 1);
    int ec;
    const double fc = log2_frac(dc, tab, ec);
    const double L = (double)(ec + eN - ea - eb) + (((fc + fN) - fa) - fb);
    return c > 0 ? dc * L : 0.0;
}

__device__ __forceinline__ double mi_exact(int g, const Marg& A, const Marg& B, int N, double dN, int eN,
                                           double fN, const double2* __restrict__ tab) {
    double s = cell_term(g, A.e1, A.f1, B.e1, B.f1, eN, fN, tab);                   // (1,1)
    s += cell_term(A.v - g, A.e1, A.f1, B.e0, B.f0, eN, fN, tab);                   // (1,0)
    s += cell_term(B.v - g, A.e0, A.f0, B.e1, B.f1, eN, fN, tab);                   // (0,1)
    s += cell_term(N - A.v - B.v + g, A.e0, A.f0, B.e0, B.f0, eN, fN, tab);         // (0,0)
    return s / dN;
}

// Epsilon mode (engine.py:112-113): p * log2((p + eps) / (e + eps)) with
// p = count / n and e = (a / n)(b / n), evaluated with the reference's operations.
__device__ __forceinline__ double mi_epsilon(int g, int vi, int vj, int N, double dN, double eps) {
    const double a1 = (double)vi, a0 = (double)(N - vi), b1 = (double)vj, b0 = (double)(N - vj);
    const double pa1 = a1 / dN, pa0 = a0 / dN, pb1 = b1 / dN, pb0 = b0 / dN;
    double p, s;
    p = (double)g / dN;                s = p * log2((p + eps) / (pa1 * pb1 + eps));
    p = (double)(vi - g) / dN;         s += p * log2((p + eps) / (pa1 * pb0 + eps));
    p = (double)(vj - g) / dN;         s += p * log2((p + eps) / (pa0 * pb1 + eps));
    p = (double)(N - vi - vj + g) / dN; s += p * log2((p + eps) / (pa0 * pb0 + eps));
    return s;
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

template <int CG>
struct TileWalk {
    // Linear walk over (my tile, k-block) pairs: step g -> tile index, k-block.
    int cluster, n_clusters, n_tiles, nkb;
    __device__ __forceinline__ bool at(long long g, int& t, int& kb) const {
        const long long it = g / nkb;
        t = cluster + (int)it * n_clusters;
        kb = (int)(g - it * nkb);
        return t < n_tiles;
    }
};

// One 32-column chunk of the epilogue for one thread (= one output row).
template <int OUT, int MODE, bool DIAG, typename T>
__device__ __forceinline__ void epilogue_chunk(const uint32_t (&r)[32], int i, int j0, const Marg& Ar,
                                               const GramMiParams& p, int eN, double fN, double dN,
                                               const double2* __restrict__ tab, T (&val)[32]) {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        const int j = j0 + k;
        const int g = (int)r[k];
        if constexpr (OUT == MI_OUT_COUNTS) {
            val[k] = g;
        } else {
            const Marg Bc = load_marg(p.colstat, j);
            // Each element is evaluated in (min, max) orientation so the two
            // halves of a diagonal tile are bit-identical mirrors.
            const bool sw = DIAG && (j < i);
            double x;
            if constexpr (MODE == MI_MODE_EXACT) {
                x = sw ? mi_exact(g, Bc, Ar, p.n_rows, dN, eN, fN, tab)
                       : mi_exact(g, Ar, Bc, p.n_rows, dN, eN, fN, tab);
            } else {
                x = mi_epsilon(g, sw ? Bc.v : Ar.v, sw ? Ar.v : Bc.v, p.n_rows, dN, p.eps);
            }
            if (DIAG && !p.include_diagonal && i == j) x = 0.0;
            val[k] = (T)x;
        }
    }
}

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
    double2* const tab = reinterpret_cast<double2*>(smem + SmemLayout::tab_off);
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
    if (threadIdx.x >= kEpiWarp0 * 32 && threadIdx.x < kEpiWarp0 * 32 + 128)
        tab[threadIdx.x - kEpiWarp0 * 32] = kLog2TabInit[threadIdx.x - kEpiWarp0 * 32];
    if (warp == 2) tmem_alloc<CG>(tmem_slot, C::TMEM_COLS);
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot_ptr;

    const int nkb = p.num_k_blocks;
    const TileWalk<CG> walk{cluster, n_clusters, p.n_tiles, nkb};

    if (warp == 0) {
        // ================= TMA producer =================
        if (lane == 0) {
            const uint64_t policy = p.l2_hint == 1   ? l2_policy_evict_last()
                                    : p.l2_hint == 2 ? l2_policy_evict_first()
                                                     : l2_policy_evict_normal();
            const int pf = p.prefetch_dist;
            const uint32_t fb_rank = (CG == 2) ? 0u : rank;  // CG == 2: signal the leader's barrier
            int s = 0;
            uint32_t ph = 0;
            // warm the L2 with the first kPrefetchDist k-blocks
            for (long long g = 0; g < pf; ++g) {
                int t, kb;
                if (!walk.at(g, t, kb)) break;
                const int2 tile = p.tiles[t];
                tma_prefetch_3d(&tmap_x, 0, tile.x * C::TS + (int)rank * 128, kb);
                tma_prefetch_3d(&tmap_x, 0, tile.y * C::TS + (int)rank * 128, kb);
            }
            int t, kb;
            for (long long g = 0; walk.at(g, t, kb); ++g) {
                const int2 tile = p.tiles[t];
                const int rowA = tile.x * C::TS + (int)rank * 128;
                const int rowB = tile.y * C::TS + (int)rank * 128;
                int tp, kbp;
                if (pf > 0 && walk.at(g + pf, tp, kbp)) {
                    const int2 tpf = p.tiles[tp];
                    tma_prefetch_3d(&tmap_x, 0, tpf.x * C::TS + (int)rank * 128, kbp);
                    tma_prefetch_3d(&tmap_x, 0, tpf.y * C::TS + (int)rank * 128, kbp);
                }
                mbar_wait(empty_bar(s), ph ^ 1u);
                const uint32_t fb = (CG == 2) ? map_to_cta(full_bar(s), fb_rank) : full_bar(s);
                if (rank == 0) mbar_arrive_expect_tx(full_bar(s), C::STAGE_TX);
                tma_load_3d<CG>(sA + s * kStageHalfBytes, &tmap_x, fb, 0, rowA, kb, policy);
                tma_load_3d<CG>(sB + s * kStageHalfBytes, &tmap_x, fb, 0, rowB, kb, policy);
                if (++s == kStages) { s = 0; ph ^= 1u; }
            }
            // drain: the last commit of every stage must land before exit
            for (int q = 0; q < kStages; ++q) {
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
        named_barrier_sync(1, kNumEpiWarps * 32);  // log2 table is in smem
        const int q = warp & 3;                    // TMEM lane quadrant of this warp
        const int h = (warp - kEpiWarp0) >> 2;     // which half of the accumulator columns
        const int row_local = q * 32 + (int)lane;
        const int m = p.m;
        const double dN = (double)p.n_rows;
        int eN;
        const double fN = log2_frac(dN, tab, eN);  // same routine as the per-column logs
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
            Marg Ar{0.0, 0.0, 0, 0, 0};
            if constexpr (OUT != MI_OUT_COUNTS) Ar = load_marg(p.colstat, i);  // colstat has m_pad rows
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
                if (diag)
                    epilogue_chunk<OUT, MODE, true>(r, i, j0, Ar, p, eN, fN, dN, tab, val);
                else
                    epilogue_chunk<OUT, MODE, false>(r, i, j0, Ar, p, eN, fN, dN, tab, val);
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
