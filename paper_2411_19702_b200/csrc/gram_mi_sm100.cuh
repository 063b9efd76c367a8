// Kernel template of the fused Gram + MI path (instantiated by gram_mi_inst_*.cu).
#pragma once
// Kernels 2+3: symmetric upper-triangle 0/1 Gram on tcgen05 with the mutual-
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
// Operand: X holds bit r of column c as an e2m1 nibble
// (FP4 = true: kind::mxf4, unit block scales, fp32 accumulators -- exact
// counts below 2^24 rows -- at twice the int8 rate) or as an int8 byte
// (kind::i8, s32 accumulators), stored k-blocked as [ld/128][m_pad][128 bytes]
// (m_pad % 256 == 0, zero padded) so each 128 x 128-byte TMA box is one
// contiguous 16 KB chunk.  Both GEMM operands are row blocks of X.
//
// Warp roles (one CTA per SM, persistent over a static tile list):
//   warp 0            TMA producer (one lane): A = X[rows of I], B = X[rows of J]
//   warp 1            TMEM allocator; then MMA issuer (one lane, leader CTA)
//   warps 2 .. 2+E-1  epilogue (E = 8): tcgen05.ld -> counts -> MI -> global
//   warp 2+E          pacer (leader CTA, PACE builds): publishes this pair's
//                     k-block progress and the minimum over all pairs
// CG == 2: a CTA pair (cluster of 2) computes a 256x256 tile with
// tcgen05.mma.cta_group::2 (M=256, N=256); each CTA stages half of A and half
// of B, and owns 128 accumulator rows.  CG == 1: 128x128 tiles on one SM
// (int8 only).  TMEM: int8 -- two accumulators (double-buffered); e2m1 -- one
// accumulator, a spare copy region and the block scales (see kSfCol below).
//
// Word-operand build (XP = true; tall-N / narrow-m): no X -- the operands are
// expanded from the packed words inside the kernel.  Roles:
//   warp 0            raw producer (one lane): TMA of packed words (16 words x
//                     128 columns per operand half) into a 2-stage raw ring
//   warp 1            MMA issuer: one warp-uniform loop over main tiles and the
//                     tail unit; diagonal tiles read B from the A stage
//   warps 2 .. 5      epilogue (E = 4); with xp_stats they first build the
//                     T table and the column statistics (grid-wide barriers)
//   warp 6            idle (the pacer slot)
//   warps 7 .. 14     expanders, two groups of 4: raw stage -> swizzled e2m1
//                     operand stages, proxy fence, relaxed arrive on the leader
// (xp_put_row / xp stats: below).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <type_traits>

#include "colstat.cuh"
#include "milog.cuh"
#include "mi_kernels.h"
#include "ptx.cuh"

namespace mib200 {

constexpr int kEpiWarp0 = 2;
constexpr int kBK = 128;                    // K bytes per pipeline stage (= 128B swizzle span)
constexpr int kStageHalfBytes = 128 * kBK;  // one 128-row operand half: 16 KB
constexpr uint32_t kMaxSmem = 232448;       // 227 KB opt-in per CTA on sm_100

template <int CG, int EW>
struct Cfg {
    static constexpr int TS = 128 * CG;             // square output tile
    static constexpr int MMA_M = 128 * CG;
    static constexpr int MMA_N = 128 * CG;
    static constexpr int ACC_COLS = MMA_N;          // TMEM columns per accumulator
    static constexpr int TMEM_COLS = 2 * ACC_COLS;  // int8: two accumulators; e2m1: one + spare + scales
    static constexpr int EPI_WARPS = EW;
    static constexpr int PACER_WARP = kEpiWarp0 + EW;
    static constexpr int THREADS = 32 * (kEpiWarp0 + EW);   // + one pacer warp when pacing
    static constexpr int COL_PARTS = EW / 4;        // epilogue warps per TMEM lane quadrant
    static constexpr int WARP_COLS = ACC_COLS / COL_PARTS;
    static constexpr uint32_t STAGE_TX = CG * 2 * kStageHalfBytes;  // bytes landing per stage
    static_assert(EW % 4 == 0 && WARP_COLS % 16 == 0, "bad epilogue split");
};

// Per-tile column marginals staged in shared memory by the epilogue: the
// FP64-path logs and the fixed-point (table path) term of each column.
struct ColS {
    double v, e1, e0, f1, f0;  // v, and log2 v = e1 + f1, log2 (N - v) = e0 + f0
    long long q;               // T(v) + T(N - v)
    int vi, pad;
};
constexpr uint32_t kTabBytes = 128u * 16u;  // log2_frac double2 table

// XP builds: a ring of raw-word stages in front of the operand ring.  One raw
// stage holds, per operand half, 128 columns x 128 bytes of packed words (16
// words = 4 k-blocks of 256 rows each: every column row is one full 128-byte
// line of the words array), loaded by TMA with the 128-byte swizzle.
constexpr int kXpRawStages = 2;
constexpr int kXpKbPerRaw = 4;                 // k-blocks per raw stage
constexpr int kXpPrefetch = 6;                 // raw stages of L2 prefetch ahead of the TMA loads
constexpr uint32_t kXpRawHalfBytes = 128 * 128;

template <int CG, int ST, bool XP = false>
struct SmemLayout {
    static constexpr uint32_t CSZ = (uint32_t)sizeof(ColS);
    static constexpr uint32_t TABB = kTabBytes;
    static constexpr int RS = XP ? kXpRawStages : 0;
    static constexpr uint32_t a_off = 0;
    static constexpr uint32_t b_off = ST * kStageHalfBytes;
    static constexpr uint32_t raw_off = 2 * ST * kStageHalfBytes;   // XP: raw stages [RS][A, B]
    static constexpr uint32_t tab_off = raw_off + RS * 2 * kXpRawHalfBytes;  // log tables
    static constexpr uint32_t col_off = tab_off + TABB;            // column stats [2][TS]
    static constexpr uint32_t bar_off = col_off + 2 * 128 * CG * CSZ;
    // full[ST], empty[ST], tfull[2], tempty[2], tmem slot, (XP) raw_full[RS], raw_empty[RS], pacing words
    static constexpr uint32_t raw_bar_off = bar_off + (2 * ST + 4) * 8 + 8;
    static constexpr uint32_t pace_off = raw_bar_off + 2 * RS * 8;
    static constexpr uint32_t bytes = pace_off + 16;
    // + alignment slack when it fits (the dynamic window is normally 1 KB aligned)
    static constexpr uint32_t request = bytes + 1024 <= kMaxSmem ? bytes + 1024 : kMaxSmem;
    static_assert(bytes <= kMaxSmem, "pipeline does not fit in shared memory");
};

// ---------------------------------------------------------------- epilogue math
//
// Exact-mode MI of one pair (engine.py:105-109,116-141), from integer counts.
// Each cell contributes c * log2(c N / (a b)), summed in the reference's fixed
// order (1,1), (1,0), (0,1), (0,0) and divided by N at the end.  The log of the
// ratio is assembled as integer exponents plus table-driven mantissa fractions
// (milog.cuh): L = ((e_c + ((e_N - e_a) - e_b)) + (((f_c + f_N) - f_a) - f_b),
// with the marginal logs precomputed once per column by kernel 1.  Identical
// mantissas cancel exactly, so an identical balanced pair gives exactly 1.0 and
// an independent one (c N == a b with equal mantissas) exactly 0.0, as in the
// reference; elsewhere the result is within ~1e-15 of the reference's value.
// All counts are exact integers held in doubles; no I2F conversions.

struct RowMarg {        // the tile row's (A side) marginals
    double v, nv;       // v_i, N - v_i
    double er1, er0;    // e_N - e(v_i), e_N - e(N - v_i)
    double f1, f0;
};

__device__ __forceinline__ RowMarg row_marg(const ColS& s, double eN, double dN) {
    return RowMarg{s.v, dN - s.v, eN - s.e1, eN - s.e0, s.f1, s.f0};
}
__device__ __forceinline__ ColS col_s(const ColStat& s) { return ColS{s.v, s.e1, s.e0, s.f1, s.f0, s.q, s.vi, 0}; }

// c * L for one cell; c == 0 contributes exactly 0 (0 * log 0 = 0).
// LOW: float32 output -- a degree-3 log polynomial (truncation < 1.3e-9
// absolute in log2 of the mantissa, 0 <= u < 2^-7; the cell weights c / N sum
// to 1, so < ~1.3e-9 in MI: far below the 1e-6 contract) instead of degree 8.
template <bool LOW = false>
__device__ __forceinline__ double cell_term(double c, double eab, double fa, double fb, double fN,
                                            const double2* __restrict__ tab) {
    // c > 0 ? c : 1 by an integer compare of the bits (c >= 0), off the FP64 pipe
    const long long cb = __double_as_longlong(c);
    const double cs = cb != 0 ? c : 1.0;
    const int hi = __double2hiint(cs);
    const int lo = __double2loint(cs);
    const double m = __hiloint2double((hi & 0x000FFFFF) | 0x3FF00000, lo);  // mantissa in [1, 2)
    const double2 t = tab[(hi >> 13) & 127];
    const double u = fma(m, t.x, -1.0);
    double p;
    if constexpr (LOW) {
        p = kLog2C3;
    } else {
        p = fma(u, kLog2C8, kLog2C7);
        p = fma(u, p, kLog2C6);
        p = fma(u, p, kLog2C5);
        p = fma(u, p, kLog2C4);
        p = fma(u, p, kLog2C3);
    }
    p = fma(u, p, kLog2C2);
    p = fma(u, p, kLog2C1);
    const double fc = fma(u, p, t.y);                                         // log2(mantissa)
    const double ec = u32_to_double((uint32_t)hi >> 20) - 1023.0;             // exponent, exact
    const double L = (ec + eab) + (((fc + fN) - fa) - fb);
    return __dmul_rn(c, L);  // explicit rounding: no FMA contraction with the running sum,
}                            // so every call site (both diagonal orientations) agrees bitwise

// s / N, correctly rounded: q = s * RN(1/N) refined by one exact-remainder step.
__device__ __forceinline__ double div_n(double s, double dN, double rN) {
    const double q = s * rN;
    const double r = fma(-q, dN, s);
    return fma(r, rN, q);
}

template <bool LOW = false>
__device__ __forceinline__ double mi_exact(double g, const RowMarg& A, const ColS& B, double fN,
                                           double dN, double rN, const double2* __restrict__ tab) {
    const double c10 = A.v - g;
    const double c01 = B.v - g;
    const double c00 = (A.nv - B.v) + g;
    double s = cell_term<LOW>(g, A.er1 - B.e1, A.f1, B.f1, fN, tab);               // (1,1)
    s = __dadd_rn(s, cell_term<LOW>(c10, A.er1 - B.e0, A.f1, B.f0, fN, tab));      // (1,0)
    s = __dadd_rn(s, cell_term<LOW>(c01, A.er0 - B.e1, A.f0, B.f1, fN, tab));      // (0,1)
    s = __dadd_rn(s, cell_term<LOW>(c00, A.er0 - B.e0, A.f0, B.f0, fN, tab));      // (0,0)
    return LOW ? s * rN : div_n(s, dN, rN);
}

// Epsilon mode (engine.py:112-113): p * log2((p + eps) / (e + eps)) with
// p = count / n and e = (a / n)(b / n), evaluated with the reference's operations.
__device__ __forceinline__ double mi_epsilon(double g, double vi, double vj, double dN, double eps) {
    const double a1 = vi, a0 = dN - vi, b1 = vj, b0 = dN - vj;
    const double pa1 = a1 / dN, pa0 = a0 / dN, pb1 = b1 / dN, pb0 = b0 / dN;
    // explicit roundings (no FMA contraction), like the reference's NumPy ops
    auto term = [&](double c, double pa, double pb) {
        const double p = c / dN;
        const double e = __dadd_rn(__dmul_rn(pa, pb), eps);
        return __dmul_rn(p, log2(__dadd_rn(p, eps) / e));
    };
    double s = term(g, pa1, pb1);
    s = __dadd_rn(s, term(vi - g, pa1, pb0));
    s = __dadd_rn(s, term(vj - g, pa0, pb1));
    s = __dadd_rn(s, term((dN - vi - vj) + g, pa0, pb0));
    return s;
}

template <int OUT>
struct OutT;
template <> struct OutT<MI_OUT_COUNTS> { using T = int32_t; };
template <> struct OutT<MI_OUT_F64> { using T = double; };
template <> struct OutT<MI_OUT_F32> { using T = float; };

__device__ __forceinline__ void store_pair(double* p, double a, double b) {
    *reinterpret_cast<double2*>(p) = make_double2(a, b);
}
__device__ __forceinline__ void store_pair(float* p, float a, float b) {
    *reinterpret_cast<float2*>(p) = make_float2(a, b);
}
__device__ __forceinline__ void store_pair(int32_t* p, int32_t a, int32_t b) {
    *reinterpret_cast<int2*>(p) = make_int2(a, b);
}

// One 32-byte store (STG.256, sm_100): a full L2 sector per thread.  The
// direct-tile stores are the epilogue's only stores that are not coalesced
// across the warp (32 rows per instruction); at 16 bytes per thread they cost
// ~6% of the MMA rate at config 3 (half-sector writes), measured with the
// debug store masks.
__device__ __forceinline__ void store32(double* p, const double* v) {
    asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(__double_as_longlong(v[0])),
                 "l"(__double_as_longlong(v[1])), "l"(__double_as_longlong(v[2])), "l"(__double_as_longlong(v[3]))
                 : "memory");
}
__device__ __forceinline__ void store32(float* p, const float* v) {
    asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(v[0]), "f"(v[1]),
                 "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}
__device__ __forceinline__ void store32(int32_t* p, const int32_t* v) {
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v[0]), "r"(v[1]),
                 "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

// Output stores with an L2 eviction-priority hint (experiments: debug bit 8 =
// evict_first for the output, so it does not push operand lines out of L2).
__device__ __forceinline__ void store32h(double* p, const double* v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.b64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p),
                 "l"(__double_as_longlong(v[0])), "l"(__double_as_longlong(v[1])), "l"(__double_as_longlong(v[2])),
                 "l"(__double_as_longlong(v[3])), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void store32h(float* p, const float* v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8}, %9;" ::"l"(p), "f"(v[0]),
                 "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void store32h(int32_t* p, const int32_t* v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8}, %9;" ::"l"(p), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void st1h(double* p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st1h(float* p, float v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st1h(int32_t* p, int32_t v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}

// The epilogue's stores of 16 finished values of row i, columns j0 .. j0+15:
// the coalesced mirror store of column i and the direct store of row i (or
// the packed upper triangle).
template <bool DIAG, typename T>
__device__ __forceinline__ void store16(const T (&v)[16], int i, int j0, const GramMiParams& p,
                                        T* __restrict__ out, int64_t ld, bool row_ok, bool vec_ok) {
    const int m = p.m;
    if (p.debug & 1) {  // keep the math alive without storing the tile
        T acc = v[0];
#pragma unroll
        for (int k = 1; k < 16; ++k) acc = acc + v[k];
        if (acc == (T)-12345) out[0] = acc;
        return;
    }
    if (!row_ok) return;
    if (ld == 0) {
        // packed upper triangle (ld_out = 0): element (i, j >= i) at
        // i m - i (i - 1) / 2 + (j - i); no mirror, nothing below the diagonal
        T* row = out + ((int64_t)i * m - ((int64_t)i * (i - 1)) / 2 - i);
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (j0 + k < m && j0 + k >= i) row[j0 + k] = v[k];
        return;
    }
    // 2) mirror tile: row j, column i (coalesced across the warp)
    const bool hint = (p.debug & 8) != 0;
    const uint64_t pol = hint ? l2_policy_evict_first() : 0ull;
    if (!DIAG && !p.tile_major && !(p.debug & 2)) {
        if (hint) {
#pragma unroll
            for (int k = 0; k < 16; ++k)
                if (j0 + k < m) st1h(out + (int64_t)(j0 + k) * ld + i, v[k], pol);
        } else {
#pragma unroll
            for (int k = 0; k < 16; ++k)
                if (j0 + k < m) out[(int64_t)(j0 + k) * ld + i] = v[k];
        }
    }
    // 3) direct tile: row i, columns j0 .. j0+15
    if (p.debug & 4) return;
    T* dst = out + (int64_t)i * ld + j0;
    if ((reinterpret_cast<uintptr_t>(dst) & 31) == 0 && j0 + 15 < m) {
        if (hint) {
#pragma unroll
            for (int k = 0; k < 16; k += 32 / (int)sizeof(T)) store32h(dst + k, v + k, pol);
        } else {
#pragma unroll
            for (int k = 0; k < 16; k += 32 / (int)sizeof(T)) store32(dst + k, v + k);
        }
        return;
    }
#pragma unroll
    for (int k = 0; k < 16; k += 2) {
        if (vec_ok && j0 + k + 1 < m) {
            store_pair(dst + k, v[k], v[k + 1]);
        } else {
            if (j0 + k < m) dst[k] = v[k];
            if (j0 + k + 1 < m) dst[k + 1] = v[k + 1];
        }
    }
}

// The tile row's fixed-point marginals (table path).
struct RowQ {
    int v, nmv;      // v_i, N - v_i
    long long kq;    // T(N) - (T(v_i) + T(N - v_i))
};

// 16 columns of one output row (this thread's TMEM lane): MI (or counts), the
// coalesced mirror store of column i and the direct store of row i.
// TABLE: exact mode through the fixed-point c log2 c table (integer sums, no
// FP64 -- B200 runs FP64 on the tensor datapath, ~23x slower under tcgen05.mma);
// otherwise the FP64 epilogue (epsilon mode, and exact-mode tiles whose column
// sums are too spread out for the table gathers to stay in L1).
// HYB (with TABLE): the hybrid path -- T(g), T(a - g), T(b - g) gathered, T(c00)
// evaluated by the table's own generating function fix_xlog2x (bit-identical to
// the entry, so exactness is unchanged): c00 = N - a - b + g is the one
// argument that scatters over the table when column sums are spread, and its
// L1 misses are what rules the full table out for such tiles.
template <int OUT, int MODE, bool DIAG, bool TABLE, bool HYB, typename T>
__device__ __forceinline__ void epilogue16(const uint32_t (&r)[16], int i, int j0, const RowMarg& A, const RowQ& AQ,
                                           const ColS* __restrict__ cols, const ColS& Arow,
                                           const GramMiParams& p, double eN, double fN, double dN, double rN,
                                           const double2* __restrict__ tab, T* __restrict__ out, int64_t ld,
                                           bool row_ok, bool vec_ok) {
    // 1) all 16 values into registers first: independent chains (and table
    //    gathers) the scheduler can overlap, no stores in between
    T v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int j = j0 + k;
        if constexpr (OUT == MI_OUT_COUNTS) {
            v[k] = (T)r[k];
        } else if constexpr (TABLE) {
            // integer sum of fixed-point terms: exact and order-independent, so
            // both halves of a diagonal tile agree bit for bit
            const int g = (int)r[k];
            const int bv = cols[k].vi;
            const long long* __restrict__ X = p.xlogx;
            const long long t00 = HYB ? fix_xlog2x((unsigned)(AQ.nmv - bv + g), p.fix_s, p.fix_r, p.fix_lg)
                                      : __ldg(X + (AQ.nmv - bv + g));
            const long long S = (__ldg(X + g) + __ldg(X + (AQ.v - g))) + (__ldg(X + (bv - g)) + t00) +
                                (AQ.kq - cols[k].q);
            T x = fixed_to_fp<T>(S, p.rcp, p.off0);
            if (DIAG && !p.include_diagonal && i == j) x = (T)0;
            v[k] = x;
        } else {
            const double g = u32_to_double(r[k]);
            const ColS& B = cols[k];
            double x;
            if constexpr (MODE == MI_MODE_EXACT) {
                if (DIAG && j < i) {
                    // (min, max) orientation: the two halves of a diagonal
                    // tile are then bit-identical mirrors
                    x = mi_exact<OUT == MI_OUT_F32>(g, row_marg(B, eN, dN), Arow, fN, dN, rN, tab);
                } else {
                    x = mi_exact<OUT == MI_OUT_F32>(g, A, B, fN, dN, rN, tab);
                }
            } else {
                x = (DIAG && j < i) ? mi_epsilon(g, B.v, A.v, dN, p.eps) : mi_epsilon(g, A.v, B.v, dN, p.eps);
            }
            if (DIAG && !p.include_diagonal && i == j) x = 0.0;
            v[k] = (T)x;
        }
    }
    store16<DIAG>(v, i, j0, p, out, ld, row_ok, vec_ok);
}

// 16 columns of one output row through the float32 epilogue (f32_mi,
// milog.cuh): FP32 pipe only, so it overlaps the next tile's MMAs.  Diagonal
// tiles evaluate (min, max) orientations so the two halves are bit-identical.
// RAW: r holds the fp32 accumulator words themselves (exact integer counts),
// else integer counts (K-split partial sums, int8 accumulators).
#ifndef MI_F32_EPI_YIELD
#define MI_F32_EPI_YIELD 1   // yield after every n-th element of the float32 epilogue (0 = never; experiments)
#endif
constexpr int kF32EpiYield = MI_F32_EPI_YIELD;
template <bool DIAG, bool RAW>
__device__ __forceinline__ void epilogue16_f32(const uint32_t (&r)[16], int i, int j0, const ColF& Af,
                                               const ColF* __restrict__ cols, const GramMiParams& p, float dN,
                                               float rN, float* __restrict__ out, int64_t ld, bool row_ok,
                                               bool vec_ok) {
    float v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const float g = RAW ? __uint_as_float(r[k]) : __uint2float_rn(r[k]);  // exact: counts < 2^24
        const int j = j0 + k;
        float x;
        if constexpr (DIAG) {
            // (min, max) orientation by selecting the operands, not the call:
            // the lanes on both sides of the diagonal share one instruction
            // stream (two calls under a per-lane condition ran both: a 151 k
            // cycle epilogue against 80 k, and a pair held up by it holds every
            // pair up through the pacing window)
            const bool sw = j < i;
            const ColF B = cols[k];
            ColF X = Af, Y = B;
            if (sw) { X = B; Y = Af; }
            x = f32_mi(g, X, Y, dN, rN);
        } else {
            x = f32_mi(g, Af, cols[k], dN, rN);
        }
        if (DIAG && !p.include_diagonal && i == j) x = 0.0f;
        v[k] = x;
        // Give the issue slot away after every element.  This epilogue is a
        // dense FP32 stream (~200 instructions per element, most of them
        // scheduled back to back with the no-yield hint), it runs beside the
        // next tile's MMAs, and its 8 warps share the 4 schedulers with the
        // producer and MMA warps, whose ~25 instructions per k-block then wait
        // behind it: without the yields the MMA pace beside a running epilogue
        // depends on how ptxas happens to pack this loop (550 to 985 cycles
        // per k-block between two builds of the same source, r02n), with them
        // it is ~515 (config 4 sustained 18.66 -> 17.93 ms).  NANOSLEEP 0 is
        // the one instruction that deschedules a warp on request.
        if constexpr (kF32EpiYield > 0) {
            if ((k + 1) % kF32EpiYield == 0) asm volatile("nanosleep.u32 0;" ::: "memory");
        }
    }
    store16<DIAG>(v, i, j0, p, out, ld, row_ok, vec_ok);
}

// ---------------------------------------------------------------- the kernel

struct TileWalk {
    // Linear walk over (my tile, k-block) pairs: step g -> tile index, k-block.
    // serp: odd tile rounds sweep K backwards, so a round starts on the
    // k-blocks the previous round read last -- still in L2 for the column
    // blocks the two rounds share.  (The MMA's accumulate flag counts steps,
    // not k-block indices, so the order of a tile's k-blocks is free: the
    // counts are exact integers either way.)
    int cluster, n_clusters, n_tiles, nkb, serp;
    __device__ __forceinline__ bool at(long long g, int& t, int& kb) const {
        const long long it = g / nkb;
        t = cluster + (int)it * n_clusters;
        const int k = (int)(g - it * nkb);
        kb = (serp & (int)it) ? nkb - 1 - k : k;
        return t < n_tiles;
    }
};

// The split tail unit's producer and MMA loops live out of line: inlined after
// the main loops they cost ~3% of the main loops' throughput (code layout).
// Operand format: FP4 = e2m1 nibbles (1.0 = 0b0010) through kind::mxf4 with
// all block scales 1.0 (E8M0 127), fp32 accumulators (exact integer counts
// below 2^24 rows), K = 256 per 128-byte k-block, at twice the kind::i8 rate
// (tools/micro/mxf4_probe.cu).  The scales take TMEM columns [496, 512) (the
// MMA reads 8 columns of them: probe), so there is room for one 256-column
// accumulator only.  To overlap the epilogue with the next tile's MMAs anyway,
// the epilogue first evacuates the accumulator -- 240 columns into the spare
// TMEM columns [256, 496), the last 16 into registers -- releases it (~10k
// cycles instead of the ~80k of the whole epilogue), then computes from there.
constexpr uint32_t kSfCol = 496;
// e2m1: consecutive accumulators alternate between TMEM columns [0, 256) and
// [kAltCol, kAltCol + 256) = [240, 496), which overlap in 16 columns only.  An
// evacuating epilogue saves those 16 columns of its tile to registers and
// releases the accumulator at once: the next tile's MMAs write the other
// position while the epilogue reads the rest of its own straight from TMEM
// (no copy: the old scheme copied 240 columns to a spare region first, ~5k
// of a config-4 tile's ~136k cycles of MMA wait).  Accumulator k of a CTA pair
// (main tiles, then the tail unit) sits at acc_col(k).
constexpr uint32_t kAltCol = 240;
__device__ __forceinline__ uint32_t acc_col(bool fp4, int k) { return (fp4 && (k & 1)) ? kAltCol : 0u; }
template <int CG, bool FP4>
__device__ __forceinline__ void mma_step(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t tmem_base, uint32_t acc) {
    if constexpr (FP4) umma_mxf4<CG>(d_tmem, adesc, bdesc, idesc, tmem_base + kSfCol, tmem_base + kSfCol, acc);
    else umma_i8<CG>(d_tmem, adesc, bdesc, idesc, acc);
}
template <int CG, bool FP4>
__host__ __device__ constexpr uint32_t mma_idesc(int M, int N) {
    return FP4 ? umma_idesc_mxf4(M, N) : umma_idesc_i8(M, N);
}
// accumulator words -> integer counts
template <bool FP4>
__device__ __forceinline__ void acc_to_counts(uint32_t (&r)[16]) {
    if constexpr (FP4) {
#pragma unroll
        for (int k = 0; k < 16; ++k) r[k] = __float2uint_rz(__uint_as_float(r[k]));
    }
}

// Tail units (GramMiParams::tail_*): column slice c (rows of B from
// J TS + c W + rank W / CG; the TMA box still moves 128 rows, the MMA reads the
// first W / CG) over k-blocks [kb0, kb1), the full K range for slices.
template <int CG, int ST>
__device__ __noinline__ uint2 producer_tail(const CUtensorMap* tmap, int2 tile, uint32_t rank, int slice, int width,
                                            int kb0, int kb1, uint32_t sA, uint32_t sB, uint32_t bar0,
                                            uint64_t policy, int s, uint32_t ph) {
    using C = Cfg<CG, 8>;
    const int rowA = tile.x * C::TS + (int)rank * 128;
    const int rowB = tile.y * C::TS + slice * width + (int)rank * (width / CG);
    for (int kb = kb0; kb < kb1; ++kb) {
        const uint32_t full = bar0 + 8u * s, empty = bar0 + 8u * (ST + s);
        mbar_wait(empty, ph ^ 1u);
        const uint32_t fb = (CG == 2) ? map_to_cta(full, 0u) : full;
        if (rank == 0) mbar_arrive_expect_tx(full, C::STAGE_TX);
        tma_load_3d<CG>(sA + s * kStageHalfBytes, tmap, fb, 0, rowA, kb, policy);
        tma_load_3d<CG>(sB + s * kStageHalfBytes, tmap, fb, 0, rowB, kb, policy);
        if (++s == ST) { s = 0; ph ^= 1u; }
    }
    return make_uint2((uint32_t)s, ph);
}

template <int CG, int ST, bool FP4>
__device__ __noinline__ void mma_tail(uint32_t tmem_base, int width, int kb0, int kb1, uint32_t sA, uint32_t sB,
                                      uint32_t bar0, int s, uint32_t ph, int acc, uint32_t aph, uint32_t acol) {
    using C = Cfg<CG, 8>;
    const uint32_t idesc = mma_idesc<CG, FP4>(C::MMA_M, width);  // M x W accumulator in columns [acol, acol + W)
    mbar_wait(bar0 + 8u * (2 * ST + 2 + acc), aph ^ 1u);  // tempty[acc]
    tc_fence_after();
    const uint32_t d_tmem = tmem_base + (uint32_t)(acc * C::ACC_COLS) + acol;
    for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(bar0 + 8u * s, ph);  // full[s]
        tc_fence_after();
        const uint64_t adesc = umma_desc_sw128_kmajor(sA + s * kStageHalfBytes);
        const uint64_t bdesc = umma_desc_sw128_kmajor(sB + s * kStageHalfBytes);
#pragma unroll
        for (int k = 0; k < kBK / 32; ++k)
            mma_step<CG, FP4>(d_tmem, adesc + 2u * k, bdesc + 2u * k, idesc, tmem_base, (kb != kb0 || k != 0) ? 1u : 0u);
        umma_commit<CG>(bar0 + 8u * (ST + s));  // empty[s]
        if (++s == ST) { s = 0; ph ^= 1u; }
    }
    umma_commit<CG>(bar0 + 8u * (2 * ST + acc));  // tfull[acc]
}

// Threads of a build: producer + MMA + epilogue warps, the pacer slot (PACE
// builds; XP builds keep the slot idle), and the XP builds' expander warps.
template <int CG, int EW, bool PACE, bool XP>
constexpr int kernel_threads() {
    return Cfg<CG, EW>::THREADS + ((PACE || XP) ? 32 : 0) + (XP ? 32 * kXpWarps : 0);
}

// XP: one step of a word-operand producer -- 32 bytes of packed words (256
// rows of one column, one k-block) -> the column's 128-byte row of the
// stage, e2m1 nibbles 0 / 1.0 (0b0010).  Bit b of 32-bit word c (rows 32c ..
// 32c + 31 of the k-block) goes to nibble 8 (b & 3) + (b >> 2) of 16-byte
// chunk c; any bijection rows -> K slots serves, as long as every column uses
// the same one (both operands are rows of X), and this one costs one shift
// and one AND per 8 nibbles.  Chunk c lands at 16-byte slot c ^ (row & 7):
// the 128-byte swizzle the UMMA descriptors (and TMA) use.  A warp's 32
// consecutive rows fill each 128-byte bank line once per store: no conflicts.
__device__ __forceinline__ void xp_put_row(uint32_t row_addr, uint32_t sw, const uint64_t (&w)[4]) {
    constexpr uint32_t M = 0x22222222u;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t x = h ? (uint32_t)(w[q] >> 32) : (uint32_t)w[q];
            const uint32_t c = (uint32_t)(2 * q + h);
            sts128(row_addr + ((c ^ sw) << 4), (x << 1) & M, x & M, (x >> 1) & M, (x >> 2) & M);
        }
    }
}
template <int CG, int OUT, int MODE, int ST, int EW, bool PACE, bool FP4, bool XP = false>
__global__ void __launch_bounds__(kernel_threads<CG, EW, PACE, XP>(), 1)
gram_mi_kernel(const __grid_constant__ CUtensorMap tmap_x, const GramMiParams p) {
    static_assert(!XP || (FP4 && CG == 2 && !PACE), "word-operand builds: e2m1 on CTA pairs, unpaced");
    using C = Cfg<CG, EW>;
    using T = typename OutT<OUT>::T;
    using L = SmemLayout<CG, ST, XP>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    const uint32_t base = (raw_addr + 1023u) & ~1023u;  // SW128 needs 1024-B alignment
    if (base - raw_addr + L::bytes > L::request) __trap();
    uint8_t* const smem = smem_raw + (base - raw_addr);

    const uint32_t sA = base + L::a_off;
    const uint32_t sB = base + L::b_off;
    const uint32_t bar0 = base + L::bar_off;
    double2* const tab = reinterpret_cast<double2*>(smem + L::tab_off);
    ColS* const colbuf = reinterpret_cast<ColS*>(smem + L::col_off);
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto empty_bar = [&](int s) { return bar0 + 8u * (ST + s); };
    auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * ST + a); };
    auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * ST + 2 + a); };
    const uint32_t tmem_slot = bar0 + 8u * (2 * ST + 4);
    volatile uint32_t* tmem_slot_ptr = reinterpret_cast<volatile uint32_t*>(smem + L::bar_off + 8 * (2 * ST + 4));
    // pacing words: [0] k-blocks issued by this pair's leader producer, [1] minimum
    // over all pairs (written by the pacer warp), [2] producer finished
    volatile uint32_t* s_pace = reinterpret_cast<volatile uint32_t*>(smem + L::pace_off);

    const int warp = threadIdx.x / 32;
    const uint32_t lane = lane_id();
    const uint32_t rank = (CG == 2) ? cluster_ctarank() : 0u;
    const int cluster = (CG == 2) ? (int)cluster_id_x() : (int)blockIdx.x;
    const int n_clusters = (CG == 2) ? (int)num_clusters_x() : (int)gridDim.x;

    // ---- one-time setup
    if (threadIdx.x == 0) {
        prefetch_tmap(&tmap_x);
        for (int s = 0; s < ST; ++s) {
            // XP: every expander warp of both CTAs arrives on the leader's full barrier
            mbar_init(full_bar(s), XP ? CG * kXpRowWarps : 1);
            mbar_init(empty_bar(s), 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull_bar(a), 1);
            mbar_init(tempty_bar(a), CG * EW);
        }
        for (int r = 0; r < L::RS; ++r) {  // XP raw ring: TMA bytes in, expander warps out
            mbar_init(base + L::raw_bar_off + 8u * r, 1);
            mbar_init(base + L::raw_bar_off + 8u * (L::RS + r), kXpWarps);
        }
        fence_mbarrier_init();
        s_pace[0] = 0u;
        s_pace[1] = 0u;
        s_pace[2] = 0u;
    }
    const int etid = (int)threadIdx.x - kEpiWarp0 * 32;  // epilogue thread id (may be < 0)
    if (etid >= 0 && etid < 128) tab[etid] = kLog2TabInit[etid];
    if (warp == 1) tmem_alloc<CG>(tmem_slot, C::TMEM_COLS);
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot_ptr;
    constexpr int NACC = FP4 ? 1 : 2;  // accumulator buffers
    if constexpr (FP4) {
        // block scales = 1.0 (E8M0 127) in TMEM columns [kSfCol, kSfCol + 16) of both CTAs
        if (etid >= 0 && etid < 4 * 32) {  // one warp per TMEM lane quadrant
            const uint32_t one[16] = {0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu,
                                      0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu,
                                      0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu};
            tmem_st_32x32b_x16(tmem_base + ((uint32_t)((warp & 3) * 32) << 16) + kSfCol, one);
            tmem_st_wait();
        }
        tc_fence_before();
        if constexpr (CG == 2) cluster_sync(); else __syncthreads();
        tc_fence_after();
    }

    const int nkb = p.num_k_blocks;
    const TileWalk walk{cluster, n_clusters, p.n_full, nkb, p.serp & 1};
    // this cluster's split tail unit, if any
    // tail tile i runs units [u0, u0 + tail_cnt[i]) (consecutive clusters)
    const int n_tail = p.tail_split > 1 ? p.n_tiles - p.n_full : 0;
    int tail_i = 0, tail_u0 = 0;
    for (; tail_i < n_tail; ++tail_i) {
        const int c = p.tail_cnt[tail_i];
        if (cluster < tail_u0 + c) break;
        tail_u0 += c;
    }
    const bool has_tail = tail_i < n_tail;
    const int tail_s = has_tail ? (int)p.tail_cnt[tail_i] : 1;  // units of this cluster's tail tile
    const int tail_t = has_tail ? p.n_full + tail_i : 0;
    const int tail_c = has_tail ? cluster - tail_u0 : 0;
    const bool tail_k = has_tail && p.tail_kmode != 0;
    // N mode: MMA slice width; K mode: full width, K range [kb0, kb1), epilogue slice tail_we
    const int tail_w = (has_tail && !tail_k) ? C::TS / tail_s : C::TS;
    const int tail_kb0 = tail_k ? (int)((long long)tail_c * nkb / tail_s) : 0;
    const int tail_kb1 = tail_k ? (int)((long long)(tail_c + 1) * nkb / tail_s) : nkb;
    const int tail_we = tail_k ? C::TS / p.tail_epi : tail_w;
    // L2 pacing: every pair walks K at the same rate over tiles drawn from a few
    // shared column blocks; kept within a window of one another, the pairs read
    // the same k-slices of those blocks close together in time, so the L2 serves
    // them once from HBM instead of once per pair (tall N overflows the L2).
    // (a separate instantiation: the check costs ~5% in the producer loop of short-K shapes)
    const bool pacing = PACE && p.pace != nullptr && p.pace_window > 0 && rank == 0 && n_clusters <= kPaceMaxClusters;
    // XP: this cluster's work as segments -- its main tiles (full K), then its
    // tail unit -- walked identically by the raw producer, the expanders and
    // the MMA warp
    const int n_main = cluster < p.n_full ? (p.n_full - 1 - cluster) / n_clusters + 1 : 0;
    const int n_seg = n_main + (has_tail ? 1 : 0);
    // segment sg: operand half rows (first column of A's and B's half), K range, B = A
    auto seg = [&](int sg, int& ra0, int& rb0, int& kb0, int& kb1, bool& share) {
        const int2 tl = p.tiles[sg < n_main ? cluster + sg * n_clusters : tail_t];
        ra0 = tl.x * C::TS + (int)rank * 128;
        if (sg < n_main) {
            rb0 = tl.y * C::TS + (int)rank * 128;
            kb0 = 0;
            kb1 = nkb;
            share = tl.x == tl.y;
        } else {
            rb0 = tl.y * C::TS + (tail_k ? 0 : tail_c * tail_w) + (int)rank * (tail_w / CG);
            kb0 = tail_kb0;
            kb1 = tail_kb1;
            share = tl.x == tl.y && tail_w == C::TS;
        }
    };

    if (warp == 0 && !XP) {
        // ================= TMA producer =================
        // The whole warp runs the loop (warp-uniform control flow: descriptors
        // and coordinates stay in uniform registers) and one elected lane
        // issues.  Under a concurrent epilogue the producer and MMA warps get
        // a fraction of their schedulers' issue slots, so the per-k-block
        // instruction path is kept short.
        const uint64_t policy = (p.l2_hint == 1 || p.l2_hint >= 3) ? l2_policy_evict_last()
                                : p.l2_hint == 2                   ? l2_policy_evict_first()
                                                                   : l2_policy_evict_normal();
        // l2_hint 3 / 4: the row-block operand (the same for every round of a
        // band) keeps evict_last, the column-block operand (new every round)
        // loads evict_first / unchanged
        const uint64_t policy_b = p.l2_hint == 3   ? l2_policy_evict_first()
                                  : p.l2_hint == 4 ? l2_policy_evict_normal()
                                                   : policy;
        const int pf = p.prefetch_dist;
        const uint32_t fb_rank = (CG == 2) ? 0u : rank;  // CG == 2: signal the leader's barrier
        int s = 0;
        uint32_t ph = 0;
        if (lane == 0) {
            for (long long g = 0; g < pf; ++g) {  // warm the L2 with the first pf k-blocks
                int t, kb;
                if (!walk.at(g, t, kb)) break;
                const int2 tile = p.tiles[t];
                tma_prefetch_3d(&tmap_x, 0, tile.x * C::TS + (int)rank * 128, kb);
                tma_prefetch_3d(&tmap_x, 0, tile.y * C::TS + (int)rank * 128, kb);
            }
        }
        bool pace_on = pacing;
        const long long win = p.pace_window;
        // tile loop outside, k-block loop inside: the tile's coordinates are
        // loaded once per tile and nothing on the per-k-block path divides or
        // touches global memory (the epilogue's stores share the LSU with
        // such loads and would stretch their latency into the MMA's supply)
        long long g = 0;
        for (int it = 0;; ++it) {
            const int t = cluster + it * n_clusters;
            if (t >= p.n_full) break;
            const int2 tile = p.tiles[t];
            const int rowA = tile.x * C::TS + (int)rank * 128;
            const int rowB = tile.y * C::TS + (int)rank * 128;
            const bool rev = (walk.serp & it) != 0;
            const bool ptrc = p.trace && cluster == 0 && it < 64;
            long long pwait = 0;
            const long long pt0 = ptrc ? clock64() : 0;
            for (int k = 0; k < nkb; ++k, ++g) {
                const int kb = rev ? nkb - 1 - k : k;
                if (PACE && pace_on && (g & 15) == 0) {
                    if (lane == 0) s_pace[0] = (uint32_t)g;
                    if (g > win) {
                        // wait (bounded: pacing is only a hint) while the slowest pair is too far behind
                        int spins = 0;
                        while ((long long)s_pace[1] + win < g) {
                            __nanosleep(64);
                            if (++spins > 20000) { pace_on = false; break; }
                        }
                    }
                    pace_on = __all_sync(0xFFFFFFFFu, pace_on);
                }
                if (pf > 0 && lane == 0) {
                    int tp, kbp;
                    if (walk.at(g + pf, tp, kbp)) {
                        const int2 tpf = p.tiles[tp];
                        tma_prefetch_3d(&tmap_x, 0, tpf.x * C::TS + (int)rank * 128, kbp);
                        tma_prefetch_3d(&tmap_x, 0, tpf.y * C::TS + (int)rank * 128, kbp);
                    }
                }
                if (ptrc) {
                    const long long w0 = clock64();
                    mbar_wait(empty_bar(s), ph ^ 1u);
                    pwait += clock64() - w0;
                } else {
                    mbar_wait(empty_bar(s), ph ^ 1u);
                }
                if (elect_one()) {
                    const uint32_t fb = (CG == 2) ? map_to_cta(full_bar(s), fb_rank) : full_bar(s);
                    if (rank == 0) mbar_arrive_expect_tx(full_bar(s), C::STAGE_TX);
                    tma_load_3d<CG>(sA + s * kStageHalfBytes, &tmap_x, fb, 0, rowA, kb, policy);
                    tma_load_3d<CG>(sB + s * kStageHalfBytes, &tmap_x, fb, 0, rowB, kb, policy_b);
                }
                __syncwarp();
                if (++s == ST) { s = 0; ph ^= 1u; }
            }
            if (ptrc && lane == 0) {
                p.trace[1280 + it * 4 + 1 + (int)rank] = pwait;  // producer waiting for free stages
                p.trace[1280 + it * 4 + 3] = clock64() - pt0;
            }
        }
        if (has_tail) {
            uint2 st = make_uint2((uint32_t)s, ph);
            if (lane == 0)
                st = producer_tail<CG, ST>(&tmap_x, p.tiles[tail_t], rank, tail_k ? 0 : tail_c, tail_w, tail_kb0,
                                           tail_kb1, sA, sB, bar0, policy, s, ph);
            s = (int)__shfl_sync(0xFFFFFFFFu, st.x, 0);
            ph = __shfl_sync(0xFFFFFFFFu, st.y, 0);
        }
        if (lane == 0) s_pace[2] = 1u;
        // drain: the last commit of every stage must land before exit
        for (int q = 0; q < ST; ++q) {
            mbar_wait(empty_bar(s), ph ^ 1u);
            if (++s == ST) { s = 0; ph ^= 1u; }
        }
    } else if (XP && warp == 1) {
        // ================= MMA issuer (XP) =================
        // One warp-uniform loop over the segments (main tiles and the tail
        // unit alike; descriptors stay in uniform registers), one elected lane
        // issues.  Diagonal tiles read B from the A stage.
        if constexpr (XP) {
            if (rank == 0) {
                const uint64_t adesc0 = umma_desc_sw128_kmajor(sA);
                const uint64_t bdesc0 = umma_desc_sw128_kmajor(sB);
                int s = 0, acc = 0;
                uint32_t ph = 0, aph = 0;
                for (int sg = 0; sg < n_seg; ++sg) {
                    int ra0, rb0, kb0, kb1;
                    bool share;
                    seg(sg, ra0, rb0, kb0, kb1, share);
                    // tail column slices: an M x W accumulator in TMEM columns [0, W)
                    const uint32_t idesc = mma_idesc<CG, FP4>(C::MMA_M, sg < n_main ? C::MMA_N : tail_w);
                    const uint64_t bd = share ? adesc0 : bdesc0;
                    mbar_wait(tempty_bar(acc), aph ^ 1u);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem_base + (uint32_t)(acc * C::ACC_COLS) + acc_col(FP4, sg);
                    for (int kb = kb0; kb < kb1; ++kb) {
                        mbar_wait(full_bar(s), ph);
                        tc_fence_after();
                        const uint64_t soff = (uint64_t)(s * (kStageHalfBytes >> 4));
                        if (elect_one()) {
                            if (!(p.debug & 16)) {
#pragma unroll
                                for (int k = 0; k < kBK / 32; ++k)
                                    mma_step<CG, FP4>(d_tmem, adesc0 + soff + 2u * k, bd + soff + 2u * k, idesc,
                                                      tmem_base, (kb != kb0 || k != 0) ? 1u : 0u);
                            }
                            umma_commit<CG>(empty_bar(s));
                        }
                        __syncwarp();
                        if (++s == ST) { s = 0; ph ^= 1u; }
                    }
                    if (elect_one()) umma_commit<CG>(tfull_bar(acc));
                    __syncwarp();
                    if (++acc == NACC) { acc = 0; aph ^= 1u; }
                }
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer =================
        // (warp-uniform loop, one elected lane issues; see the producer)
        if (rank == 0) {
            constexpr uint32_t idesc = mma_idesc<CG, FP4>(C::MMA_M, C::MMA_N);
            // stage s's descriptors: base + s * 16 KB (address field in 16-byte units)
            const uint64_t adesc0 = umma_desc_sw128_kmajor(sA);
            const uint64_t bdesc0 = umma_desc_sw128_kmajor(sB);
            int s = 0;
            uint32_t ph = 0;
            int acc = 0;
            uint32_t aph = 0;
            int it = 0;
            for (int t = cluster; t < p.n_full; t += n_clusters, ++it) {
                mbar_wait(tempty_bar(acc), aph ^ 1u);
                tc_fence_after();
                const bool trc = p.trace && cluster == 0 && it < 64;
                if (trc && lane == 0) p.trace[it * 4 + 0] = clock64();
                const uint32_t d_tmem = tmem_base + (uint32_t)(acc * C::ACC_COLS) + acc_col(FP4, it);
                long long wait_cyc = 0;
                for (int kb = 0; kb < nkb; ++kb) {
                    if (trc) {
                        const long long w0 = clock64();
                        mbar_wait(full_bar(s), ph);
                        wait_cyc += clock64() - w0;
                    } else {
                        mbar_wait(full_bar(s), ph);
                    }
                    tc_fence_after();
                    const uint64_t soff = (uint64_t)(s * (kStageHalfBytes >> 4));
                    const uint64_t adesc = adesc0 + soff;
                    const uint64_t bdesc = bdesc0 + soff;
                    if (elect_one()) {
                        if (!(p.debug & 16)) {  // debug 16: data movement only (no MMAs)
#pragma unroll
                            for (int k = 0; k < kBK / 32; ++k) {
                                // advance 32 bytes (one K=32 int8 step) inside the swizzle atom
                                mma_step<CG, FP4>(d_tmem, adesc + 2u * k, bdesc + 2u * k, idesc, tmem_base,
                                                  (kb | k) != 0 ? 1u : 0u);
                            }
                        }
                        umma_commit<CG>(empty_bar(s));  // frees the smem slot (both CTAs)
                    }
                    __syncwarp();
                    if (++s == ST) { s = 0; ph ^= 1u; }
                }
                if (elect_one()) umma_commit<CG>(tfull_bar(acc));  // accumulator ready (both CTAs)
                __syncwarp();
                if (trc && lane == 0) {
                    p.trace[it * 4 + 1] = clock64();
                    p.trace[1280 + it * 4 + 0] = wait_cyc;  // MMA starved of operands
                }
                if (++acc == NACC) { acc = 0; aph ^= 1u; }
            }
            if (has_tail && lane == 0)
                mma_tail<CG, ST, FP4>(tmem_base, tail_w, tail_kb0, tail_kb1, sA, sB, bar0, s, ph, acc, aph,
                                      acc_col(FP4, it));
        }
    } else if (XP && (warp == 0 || warp >= C::PACER_WARP)) {
        // ================= word operands (XP) =================
        // warp 0 (one lane): TMA of raw packed words -- per operand half, 128
        //   columns x 16 words (4 k-blocks) -- into the raw ring (this CTA's
        //   barriers; each CTA loads its own halves);
        // warps PACER_WARP + 1 .. + kXpWarps (expanders): thread xt owns row xt
        //   of the CTA's halves of A and B; per k-block it reads its 32 bytes
        //   of words from the raw stage, writes the swizzled e2m1 rows
        //   (xp_put_row), fences them into the async proxy and arrives (one
        //   lane per warp) on the leader CTA's full barrier.  The expanders
        //   have no global loads in flight at that fence (TMA brings the
        //   words), so it costs a shared-memory drain, not a DRAM latency.
        // The pacer slot idles.  Diagonal tiles stage one copy (B = A).
        if constexpr (XP) {
            auto xwait = [&](uint32_t bar, uint32_t par) { mbar_wait(bar, par); };
            // experiments: per-phase cycle sums of cluster 0 (tools/xp_probe.py --trace)
            long long* const xtr = (p.trace && cluster == 0) ? p.trace + 2048 : nullptr;
            const uint32_t raw0 = base + L::raw_off;
            const uint32_t rbar0 = base + L::raw_bar_off;
            auto raw_full = [&](int r) { return rbar0 + 8u * r; };
            auto raw_empty = [&](int r) { return rbar0 + 8u * (L::RS + r); };
            auto raw_a = [&](int r) { return raw0 + (uint32_t)r * 2u * kXpRawHalfBytes; };
            if (warp == 0) {
                const uint64_t policy = p.l2_hint == 1   ? l2_policy_evict_last()
                                        : p.l2_hint == 2 ? l2_policy_evict_first()
                                                         : l2_policy_evict_normal();
                int r = 0;
                uint32_t rph = 0;
                long long pw = 0;
                for (int sg = 0; sg < n_seg; ++sg) {
                    int ra0, rb0, kb0, kb1;
                    bool share;
                    seg(sg, ra0, rb0, kb0, kb1, share);
                    const int qlast = (kb1 - 1) / kXpKbPerRaw;
                    // L2 prefetch of the raw boxes kXpPrefetch stages ahead: the raw ring
                    // holds only kXpRawStages x 4 k-blocks, less than a DRAM round trip
                    for (int q = kb0 / kXpKbPerRaw; q < min(qlast + 1, kb0 / kXpKbPerRaw + kXpPrefetch); ++q)
                        if (elect_one()) {
                            tma_prefetch_2d(&tmap_x, 4 * kXpKbPerRaw * q, ra0);
                            if (!share) tma_prefetch_2d(&tmap_x, 4 * kXpKbPerRaw * q, rb0);
                        }
                    for (int q = kb0 / kXpKbPerRaw; q <= qlast; ++q) {
                        if (q + kXpPrefetch <= qlast && elect_one()) {
                            tma_prefetch_2d(&tmap_x, 4 * kXpKbPerRaw * (q + kXpPrefetch), ra0);
                            if (!share) tma_prefetch_2d(&tmap_x, 4 * kXpKbPerRaw * (q + kXpPrefetch), rb0);
                        }
                        __syncwarp();
                        const long long c0 = xtr ? clock64() : 0;
                        xwait(raw_empty(r), rph ^ 1u);
                        if (xtr) pw += clock64() - c0;
                        if (p.debug & 64) {  // experiments: no word loads (expander throughput alone)
                            if (elect_one()) mbar_arrive_local(raw_full(r));
                        } else if (elect_one()) {
                            mbar_arrive_expect_tx(raw_full(r), (share ? 1u : 2u) * kXpRawHalfBytes);
                            tma_load_2d_local(raw_a(r), &tmap_x, raw_full(r), 4 * kXpKbPerRaw * q, ra0, policy);
                            if (!share)
                                tma_load_2d_local(raw_a(r) + kXpRawHalfBytes, &tmap_x, raw_full(r),
                                                  4 * kXpKbPerRaw * q, rb0, policy);
                        }
                        __syncwarp();
                        if (++r == L::RS) { r = 0; rph ^= 1u; }
                    }
                }
                if (xtr && lane == 0) xtr[24 + rank] = pw;
            } else if (warp > C::PACER_WARP) {
                // Two groups of kXpRowWarps warps: within each raw stage (4
                // k-blocks), group 0 expands the first two k-blocks and group 1
                // the last two, so two batches are in flight per row and every
                // scheduler runs two expander warps.  Operand stage of a k-block
                // = its position in this CTA's k-block sequence modulo ST.
                const int xw = warp - C::PACER_WARP - 1;
                const int grp = xw / kXpRowWarps;
                const int m_real = p.m;
                const int xt = (xw % kXpRowWarps) * 32 + (int)lane;
                const uint32_t full_leader0 = map_to_cta(full_bar(0), 0u);
                const uint32_t sw = (uint32_t)xt & 7u;
                int r = 0;
                uint32_t rph = 0;
                long long ctr = 0;  // k-blocks of this CTA's sequence before the current raw stage
                long long acc_t[6] = {0, 0, 0, 0, 0, 0};  // experiments (xtr): phase cycle sums
                for (int sg = 0; sg < n_seg; ++sg) {
                    int ra0, rb0, kb0, kb1;
                    bool share;
                    seg(sg, ra0, rb0, kb0, kb1, share);
                    // statistics mode: diagonal units count their columns' ones
                    const bool count = p.xp_stats && share;
                    uint32_t ones = 0;
                    for (int q = kb0 / kXpKbPerRaw; q <= (kb1 - 1) / kXpKbPerRaw; ++q) {
                        const int lo = max(kb0, q * kXpKbPerRaw), hi = min(kb1, (q + 1) * kXpKbPerRaw);
                        const int my0 = max(lo, q * kXpKbPerRaw + 2 * grp), my1 = min(hi, q * kXpKbPerRaw + 2 * grp + 2);
                        const long long c0 = xtr ? clock64() : 0;
                        xwait(raw_full(r), rph);
                        if (xtr) acc_t[0] += clock64() - c0;
                        if (my1 > my0) {
                            const bool two = my1 - my0 == 2;
                            const long long cA = ctr + (my0 - lo);
                            const int s0 = (int)(cA % ST), s1 = (int)((cA + 1) % ST);
                            const uint32_t p0 = (uint32_t)((cA / ST) & 1), p1 = (uint32_t)(((cA + 1) / ST) & 1);
                            const long long t0 = xtr ? clock64() : 0;
                            // k-block j's 32 bytes: logical chunks 2j, 2j + 1 of the swizzled 128-byte row
                            const uint32_t j = (uint32_t)(my0 - q * kXpKbPerRaw);
                            const uint32_t rowa = raw_a(r) + (uint32_t)xt * 128u;
                            uint64_t wa[2][4], wb[2][4];
#pragma unroll
                            for (int i = 0; i < 2; ++i) {
                                if (i == 0 || two) {
                                    const uint32_t jj = j + (uint32_t)i;
                                    lds128(rowa + (((2u * jj) ^ sw) << 4), wa[i][0], wa[i][1]);
                                    lds128(rowa + (((2u * jj + 1u) ^ sw) << 4), wa[i][2], wa[i][3]);
                                    if (!share) {
                                        lds128(rowa + kXpRawHalfBytes + (((2u * jj) ^ sw) << 4), wb[i][0], wb[i][1]);
                                        lds128(rowa + kXpRawHalfBytes + (((2u * jj + 1u) ^ sw) << 4), wb[i][2], wb[i][3]);
                                    }
                                }
                            }
                            if (count) {
#pragma unroll
                                for (int i = 0; i < 2; ++i)
                                    if (i == 0 || two)
                                        ones += __popcll(wa[i][0]) + __popcll(wa[i][1]) + __popcll(wa[i][2]) +
                                                __popcll(wa[i][3]);
                            }
                            const long long t1 = xtr ? clock64() : 0;
                            xwait(empty_bar(s0), p0 ^ 1u);
                            if (two) xwait(empty_bar(s1), p1 ^ 1u);
                            const long long t2 = xtr ? clock64() : 0;
                            if (!(p.debug & 32)) {  // experiments: 32 = no expansion (load pipeline alone)
#pragma unroll
                                for (int i = 0; i < 2; ++i) {
                                    if (i == 0 || two) {
                                        const uint32_t so = (uint32_t)(i ? s1 : s0) * kStageHalfBytes + (uint32_t)xt * 128u;
                                        xp_put_row(sA + so, sw, wa[i]);
                                        if (!share) xp_put_row(sB + so, sw, wb[i]);
                                    }
                                }
                            }
                            const long long t3 = xtr ? clock64() : 0;
                            // Publish: the proxy fence drains this thread's shared-memory writes
                            // (MEMBAR.CTA) and makes them visible to the async proxy; the arrives
                            // that follow are relaxed.  A release.cluster arrive would add a
                            // GPU-wide drain per warp and batch (~800 cycles measured; the
                            // pipeline is latency-bound: tools/xp_probe.py), and the data are
                            // already in this SM's shared memory when the arrive lands.
                            fence_proxy_async_smem();
                            __syncwarp();
                            if (lane == 0) {
                                mbar_arrive_cluster_relaxed(full_leader0 + 8u * s0);
                                if (two) mbar_arrive_cluster_relaxed(full_leader0 + 8u * s1);
                            }
                            if (xtr) {
                                acc_t[1] += t1 - t0;           // LDS
                                acc_t[2] += t2 - t1;           // waiting for free stages
                                acc_t[3] += t3 - t2;           // expand + STS
                                acc_t[4] += clock64() - t3;    // fence + arrive
                                acc_t[5] += two ? 2 : 1;       // k-blocks
                            }
                        }
                        __syncwarp();
                        if (lane == 0) mbar_arrive_local(raw_empty(r));  // both groups are done with it
                        if (++r == L::RS) { r = 0; rph ^= 1u; }
                        ctr += hi - lo;
                    }
                    if (count) {  // publish this warp's counts of the segment (its k-blocks, its rows)
                        if (ra0 + xt < m_real && ones) atomicAdd(&p.colstat_w[ra0 + xt].vi, (int)ones);
                        __threadfence();
                        __syncwarp();
                        if (lane == 0) atomicAdd(p.xp_sync, 1u);
                    }
                }
                if (xtr && xw == 0 && lane == 0)
                    for (int k = 0; k < 6; ++k) xtr[8 * rank + k] = acc_t[k];
                // drain: the last commit of every stage must land before exit
                if (xw == 0) {
                    for (int q = 0; q < ST; ++q, ++ctr) xwait(empty_bar((int)(ctr % ST)), (uint32_t)(((ctr / ST) & 1) ^ 1));
                }
            }
        }
    } else if (PACE && warp == C::PACER_WARP) {
        // ================= pacer =================
        if (pacing) {
            volatile uint32_t* gp = p.pace;
            if (lane == 0) gp[cluster * kPaceStride] = 0u;
            uint32_t last = 0u;
            for (;;) {
                const uint32_t done = s_pace[2];
                const uint32_t mine = s_pace[0];
                if (lane == 0 && mine != last) {
                    gp[cluster * kPaceStride] = mine;
                    last = mine;
                }
                uint32_t v = 0xFFFFFFFFu;
                for (int c = (int)lane; c < n_clusters; c += 32) v = min(v, gp[c * kPaceStride]);
                v = __reduce_min_sync(0xFFFFFFFFu, v);
                if (lane == 0) s_pace[1] = v;
                if (done) break;
                __nanosleep(256);
            }
            if (lane == 0) gp[cluster * kPaceStride] = 0xFFFFFFFFu;  // finished pairs never hold others back
        }
    } else {
        // ================= epilogue =================
        if constexpr (XP) {
            if (p.xp_stats) {
                // statistics mode: while the units run, build the T table, then wait
                // for the diagonal units' column counts, write the column statistics
                // (a slice per thread across the grid) and meet every CTA at a
                // grid-wide barrier (all CTAs are co-resident: one per SM)
                const long long gtid = (long long)blockIdx.x * (EW * 32) + etid;
                const long long gthreads = (long long)gridDim.x * (EW * 32);
                if (p.xlogx_w)
                    for (long long c = gtid; c <= p.n_rows; c += gthreads)
                        p.xlogx_w[c] = fix_xlog2x((unsigned)c, p.fix_s, kFixR, kFixLG);
                volatile unsigned int* sync = p.xp_sync;
                if (etid == 0) {
                    // completions to wait for: every expander warp of every diagonal tile's units
                    unsigned int expect = 0;
                    for (int i = 0; i < n_tail; ++i) {
                        const int2 tl = p.tiles[p.n_full + i];
                        if (tl.x == tl.y) expect += p.tail_cnt[i];
                    }
                    expect *= (unsigned)(CG * kXpWarps);
                    const long long t0 = clock64();
                    while (sync[0] < expect) {
                        __nanosleep(256);
                        if (clock64() - t0 > (1ll << 36)) __trap();  // a lost unit is a bug
                    }
                    __threadfence();
                }
                named_barrier_sync(5, EW * 32);
                const int64_t m_pad = (int64_t)((p.m + C::TS - 1) / C::TS) * C::TS;
                for (long long c = gtid; c < m_pad; c += gthreads)  // whole warps: m_pad, gthreads are multiples of 32
                    write_colstat(c, (uint32_t)__ldcg(&p.colstat_w[c].vi), p.n_rows, c < p.m, p.fix_s, p.colsum,
                                  p.colstat_w, p.blkrange_w);
                __threadfence();
                named_barrier_sync(5, EW * 32);
                if (etid == 0) {
                    atomicAdd(p.xp_sync + 1, 1u);
                    const long long t0 = clock64();
                    while (sync[1] < gridDim.x) {
                        __nanosleep(256);
                        if (clock64() - t0 > (1ll << 36)) __trap();
                    }
                    __threadfence();
                }
                named_barrier_sync(5, EW * 32);
            }
        }
        const int q = warp & 3;                          // TMEM lane quadrant of this warp
        const int part = (warp - kEpiWarp0) >> 2;        // which column slice of the accumulator
        const int row_local = q * 32 + (int)lane;
        const int m = p.m;
        const double dN = (double)p.n_rows;
        const double rN = 1.0 / dN;
        const float dNf = (float)p.n_rows;           // float32 path (N < 2^24: exact)
        const float rNf = (float)rN;
        named_barrier_sync(1, EW * 32);                  // log2 table is in smem
        int eNi;
        const double fN = log2_frac(dN, tab, eNi);       // same routine as the per-column logs
        const double eN = (double)eNi;
        const bool have_table = MODE == MI_MODE_EXACT && p.xlogx != nullptr;
        const long long nln = have_table ? p.xlogx[p.n_rows] : 0ll;  // T(N) = N log2 N 2^s
        const int64_t ld = p.ld_out;
        T* __restrict__ out = reinterpret_cast<T*>(p.out);
        const uint32_t tempty_leader0 = (CG == 2) ? map_to_cta(tempty_bar(0), 0) : tempty_bar(0);
        const uint32_t tempty_leader1 = (CG == 2) ? map_to_cta(tempty_bar(1), 0) : tempty_bar(1);
        int acc = 0;
        uint32_t aph = 0;
        int it = 0;
        const bool tracer = p.trace && cluster == 0 && rank == 0 && warp == kEpiWarp0 && lane == 0;
        // one tile's epilogue, or of one column slice [c0, c0 + W) of a split
        // tail tile: N mode -- the slice's accumulator in TMEM columns [0, W);
        // K mode -- this unit's full-width partial plus the other units' ones
        int cpar = 0;
        auto epi_tile = [&](const int t, auto tail_tag) {
            constexpr int TAIL = decltype(tail_tag)::value;  // 0 whole tile, 1 N slice, 2 K-split owner
            const int c0 = TAIL ? tail_c * tail_we : 0;       // first tile column of this epilogue
            const int tc0 = TAIL == 2 ? c0 : 0;                // its accumulator column
            const int part_cols = TAIL ? tail_we / C::COL_PARTS : C::WARP_COLS;
            const int2 tile = p.tiles[t];
            const bool diag = tile.x == tile.y;
            const int i = tile.x * C::TS + (int)rank * 128 + row_local;
            // this tile's column marginals, double-buffered by tile parity: a fast
            // warp stages the next tile's while slow ones still read this one
            ColS* const cols = colbuf + cpar * C::TS;
            cpar ^= 1;
            ColS Arow{};
            RowQ AQ{0, 0, 0};
            ColF Af{};
            ColF* const colsf = reinterpret_cast<ColF*>(cols);  // the float32 path's staging (same buffer)
            bool use_table = false, use_hybrid = false, use_f32 = false;
            if constexpr (OUT != MI_OUT_COUNTS) {
                // per-tile choice (identical in both CTAs of a pair): table path
                // when the tile's column sums are clustered enough for the
                // gathers to hit in L1; otherwise the float32 epilogue for
                // float32 output, else FP64
                if (have_table) {
                    const int bl = C::TS / 128;
                    int lo = 0x7FFFFFFF, hi = -1, spread = 0;
                    for (int q2 = 0; q2 < bl; ++q2) {
                        const int2 a = p.blkrange[tile.x * bl + q2];
                        lo = min(lo, a.x);
                        hi = max(hi, a.y);
                    }
                    spread = hi >= lo ? hi - lo : 0;
                    lo = 0x7FFFFFFF;
                    hi = -1;
                    for (int q2 = 0; q2 < bl; ++q2) {
                        const int2 a = p.blkrange[tile.y * bl + q2];
                        lo = min(lo, a.x);
                        hi = max(hi, a.y);
                    }
                    spread += hi >= lo ? hi - lo : 0;
                    use_table = spread <= p.table_thr;
                }
                use_f32 = OUT == MI_OUT_F32 && MODE == MI_MODE_EXACT && p.f32_epi && !use_table;
                use_hybrid = have_table && !use_table && !use_f32 && p.hybrid;
                if (use_f32) {
                    for (int e = etid; e < C::TS; e += EW * 32) colsf[e] = p.colstat[tile.y * C::TS + e].f;
                    named_barrier_sync(2, EW * 32);
                    Af = p.colstat[i].f;
                } else {
                    for (int e = etid; e < C::TS; e += EW * 32) cols[e] = col_s(p.colstat[tile.y * C::TS + e]);
                    named_barrier_sync(2, EW * 32);
                    Arow = col_s(p.colstat[i]);  // colstat has m_pad entries
                    AQ = RowQ{Arow.vi, p.n_rows - Arow.vi, nln - Arow.q};
                }
            }
            const RowMarg A = row_marg(Arow, eN, dN);
            const bool row_ok = i < m;
            // output base: the matrix, or (tile-major shards) slot t of TS x TS
            // rows, addressed with the tile's global (i, j) so the stores are shared
            T* const o = p.tile_major ? out + ((int64_t)t * C::TS - (int64_t)tile.x * C::TS) * C::TS -
                                            (int64_t)tile.y * C::TS
                                      : out;
            const int64_t ldd = p.tile_major ? (int64_t)C::TS : ld;
            mbar_wait(tfull_bar(acc), aph);
            tc_fence_after();
            if (tracer && it < 64) p.trace[it * 4 + 2] = clock64();
            const uint32_t lane_q = (uint32_t)(q * 32) << 16;
            // Evacuate only when the epilogue is FP64-free: an FP64 epilogue next to
            // running MMAs is throttled ~23x (r01_micro.md), so FP64-path tiles keep
            // the accumulator until done and run their epilogue alone.
            const bool EVAC = FP4 && TAIL == 0 && p.evac != 0 &&
                              (OUT == MI_OUT_COUNTS || use_table || use_hybrid || use_f32 || p.evac == 2);
            // this accumulator's TMEM columns, and (EVAC) the 16 of them the next
            // accumulator overlaps (acc_col): saved here before the release
            const uint32_t accb = acc_col(FP4, it);
            const int ovl = accb ? 0 : C::TS - 16;
            uint32_t keep[16];
            if (EVAC) {
                if (ovl >= part * part_cols && ovl < (part + 1) * part_cols) {
                    tmem_ld_32x32b_x16(tmem_base + lane_q + accb + (uint32_t)ovl, keep);
                    tmem_ld_wait(keep);
                }
                // the accumulator is free: the next tile's MMAs start now (on the
                // other position)
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(tempty_leader0);
            }
#pragma unroll 1
            for (int c = 0; c < part_cols; c += 16) {
                const int col0 = part * part_cols + c;   // accumulator column
                const int j0 = tile.y * C::TS + c0 + col0;
                uint32_t r[16];
                if (EVAC && col0 == ovl) {
#pragma unroll
                    for (int k = 0; k < 16; ++k) r[k] = keep[k];
                } else {
                    tmem_ld_32x32b_x16(tmem_base + lane_q + accb + (uint32_t)(acc * C::ACC_COLS + tc0 + col0), r);
                    tmem_ld_wait(r);
                }
                if (!(FP4 && use_f32 && TAIL != 2)) acc_to_counts<FP4>(r);  // (the f32 path reads fp32 counts as is)
                if constexpr (TAIL == 2) {  // + the other K ranges (integer adds: exact in any order)
                    const size_t off = ((size_t)((tc0 + col0) / 16) * 128 + row_local) * 16;
                    // kTailSumDepth partials in flight per step (a unit sums up to ~74 of them)
#pragma unroll 1
                    for (int w0 = 0; w0 < tail_s; w0 += kTailSumDepth) {
                        uint4 x[kTailSumDepth][4];
#pragma unroll
                        for (int j = 0; j < kTailSumDepth; ++j) {
                            const int w = w0 + j;
                            const bool use = w < tail_s && w != tail_c;
                            const uint4* src = reinterpret_cast<const uint4*>(
                                p.tail_part + (size_t)((tail_u0 + (use ? w : 0)) * CG + (int)rank) * 128 * C::TS + off);
#pragma unroll
                            for (int k4 = 0; k4 < 4; ++k4) x[j][k4] = use ? __ldcg(src + k4) : make_uint4(0u, 0u, 0u, 0u);
                        }
#pragma unroll
                        for (int j = 0; j < kTailSumDepth; ++j)
#pragma unroll
                            for (int k4 = 0; k4 < 4; ++k4) {
                                r[4 * k4 + 0] += x[j][k4].x;
                                r[4 * k4 + 1] += x[j][k4].y;
                                r[4 * k4 + 2] += x[j][k4].z;
                                r[4 * k4 + 3] += x[j][k4].w;
                            }
                    }
                }
                const bool vec_ok = ((reinterpret_cast<uintptr_t>(o + (int64_t)i * ldd + j0) & (2 * sizeof(T) - 1)) == 0);
                if (use_f32) {
                    if constexpr (MODE == MI_MODE_EXACT && OUT == MI_OUT_F32) {
                        constexpr bool RAW = FP4 && TAIL != 2;
                        if (diag)
                            epilogue16_f32<true, RAW>(r, i, j0, Af, colsf + c0 + col0, p, dNf, rNf, o, ldd, row_ok,
                                                      vec_ok);
                        else
                            epilogue16_f32<false, RAW>(r, i, j0, Af, colsf + c0 + col0, p, dNf, rNf, o, ldd, row_ok,
                                                       vec_ok);
                    }
                } else if (use_table) {
                    if constexpr (MODE == MI_MODE_EXACT && OUT != MI_OUT_COUNTS) {
                        if (diag)
                            epilogue16<OUT, MODE, true, true, false>(r, i, j0, A, AQ, cols + c0 + col0, Arow, p, eN, fN,
                                                                     dN, rN, tab, o, ldd, row_ok, vec_ok);
                        else
                            epilogue16<OUT, MODE, false, true, false>(r, i, j0, A, AQ, cols + c0 + col0, Arow, p, eN, fN,
                                                                      dN, rN, tab, o, ldd, row_ok, vec_ok);
                    }
                } else if (use_hybrid) {
                    if constexpr (MODE == MI_MODE_EXACT && OUT != MI_OUT_COUNTS) {
                        if (diag)
                            epilogue16<OUT, MODE, true, true, true>(r, i, j0, A, AQ, cols + c0 + col0, Arow, p, eN, fN,
                                                                    dN, rN, tab, o, ldd, row_ok, vec_ok);
                        else
                            epilogue16<OUT, MODE, false, true, true>(r, i, j0, A, AQ, cols + c0 + col0, Arow, p, eN, fN,
                                                                     dN, rN, tab, o, ldd, row_ok, vec_ok);
                    }
                } else if (diag) {
                    epilogue16<OUT, MODE, true, false, false>(r, i, j0, A, AQ, cols + c0 + col0, Arow, p, eN, fN, dN, rN,
                                                              tab, o, ldd, row_ok, vec_ok);
                } else {
                    epilogue16<OUT, MODE, false, false, false>(r, i, j0, A, AQ, cols + c0 + col0, Arow, p, eN, fN, dN, rN,
                                                               tab, o, ldd, row_ok, vec_ok);
                }
            }
            // hand the accumulator back to the MMA warp (EVAC: done above)
            if (tracer && it < 64) p.trace[it * 4 + 3] = clock64();
            if (!EVAC) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(acc == 0 ? tempty_leader0 : tempty_leader1);
            }
            if (p.row_done) {
                // publish: this CTA's rows and mirrors of tile (I, J) are in memory
                __threadfence_system();
                named_barrier_sync(3, EW * 32);
                if (etid == 0) atomicAdd_system(p.row_done + tile.x, 1u);
            }
            if (++acc == NACC) { acc = 0; aph ^= 1u; }
        };
        // per-cluster timeline (globaltimer ns): start, main tiles done, tail done
        long long* const ctrace = (p.trace && rank == 0 && etid == 0) ? p.trace + 256 + cluster * 4 : nullptr;
        if (ctrace) ctrace[0] = (long long)global_ns();
        for (int t = cluster; t < p.n_full; t += n_clusters, ++it) epi_tile(t, std::integral_constant<int, 0>{});
        if (ctrace) ctrace[1] = (long long)global_ns();
        if (has_tail && !tail_k) {
            epi_tile(tail_t, std::integral_constant<int, 1>{});
        } else if (has_tail) {
            // K-split unit: publish the partial accumulator (all columns) ...
            mbar_wait(tfull_bar(acc), aph);
            tc_fence_after();
            uint32_t* dst_base = p.tail_part + (size_t)(cluster * CG + (int)rank) * 128 * C::TS;
#pragma unroll 1
            for (int c = 0; c < C::WARP_COLS; c += 16) {
                const int col0 = part * C::WARP_COLS + c;
                uint32_t r[16];
                tmem_ld_32x32b_x16(tmem_base + ((uint32_t)(q * 32) << 16) + acc_col(FP4, it) +
                                       (uint32_t)(acc * C::ACC_COLS + col0), r);
                tmem_ld_wait(r);
                acc_to_counts<FP4>(r);
                uint4* dst = reinterpret_cast<uint4*>(dst_base + ((size_t)(col0 / 16) * 128 + row_local) * 16);
#pragma unroll
                for (int k4 = 0; k4 < 4; ++k4)
                    __stcg(dst + k4, make_uint4(r[4 * k4], r[4 * k4 + 1], r[4 * k4 + 2], r[4 * k4 + 3]));
            }
            __threadfence();
            named_barrier_sync(4, EW * 32);
            unsigned int* flag = p.tail_flag + (tail_t - p.n_full) * 2 + rank;
            if (etid == 0) atomicAdd(flag, 1u);
            if (tail_c < p.tail_epi) {
                // ... then, as an epilogue unit, wait for every unit's partial and
                // finish column slice tail_c on the sum
                if (etid == 0) {
                    volatile unsigned int* f = flag;
                    const long long t0 = clock64();
                    while (*f < (unsigned int)tail_s) {
                        __nanosleep(64);
                        if (clock64() - t0 > (1ll << 36)) __trap();  // ~30 s: a lost unit is a bug
                    }
                    __threadfence();
                }
                named_barrier_sync(4, EW * 32);
                epi_tile(tail_t, std::integral_constant<int, 2>{});
            } else {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(acc == 0 ? tempty_leader0 : tempty_leader1);
            }
        }
        if (ctrace) ctrace[2] = (long long)global_ns();
    }

    // ---- teardown
    __syncwarp();
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc<CG>(tmem_base, C::TMEM_COLS);
}

// ---------------------------------------------------------------- launch

template <int CG, int OUT, int MODE, int ST, int EW, bool PACE, bool FP4, bool XP = false>
cudaError_t launch_impl(const CUtensorMap& tmap, const GramMiParams& p, int num_sms, cudaStream_t stream) {
    auto kern = gram_mi_kernel<CG, OUT, MODE, ST, EW, PACE, FP4, XP>;
    constexpr uint32_t smem = SmemLayout<CG, ST, XP>::request;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int max_clusters = num_sms / CG;
    int clusters = p.n_tiles < max_clusters ? p.n_tiles : max_clusters;
    if (p.tail_split > 1) {  // the host sized n_full as a multiple of max_clusters
        int units = 0;
        for (int i = 0; i < p.n_tiles - p.n_full; ++i) units += p.tail_cnt[i];
        if (p.n_full % max_clusters != 0 || p.n_tiles - p.n_full > kTailMaxUnits || units != p.tail_units ||
            units > max_clusters)
            return cudaErrorInvalidValue;
        clusters = p.n_full > 0 ? max_clusters : units;
    }
    if (clusters < 1) clusters = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(clusters * CG, 1, 1);
    cfg.blockDim = dim3(kernel_threads<CG, EW, PACE, XP>(), 1, 1);
    cfg.dynamicSmemBytes = smem;
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

}  // namespace mib200
