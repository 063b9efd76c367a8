// Per-column statistics of the fused epilogue (shared by kernel 1 and the
// word-operand build, which computes them inside the fused launch).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "milog.cuh"

namespace mib200 {

// Per-column statistics for the fused epilogue (lane/thread owning column c).
__device__ __forceinline__ void write_colstat(int64_t c, uint32_t cnt, int64_t n_rows, bool real, int fix_s,
                                              int32_t* __restrict__ colsum, ColStat* __restrict__ colstat,
                                              int2* __restrict__ blkrange) {
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
    // float32 epilogue factors: N / a and 1 / a as float pairs (1.0 for a = 0)
    const double dn = (double)n_rows;
    auto split = [](double x, float& hi, float& lo) {
        hi = (float)x;
        lo = (float)(x - (double)hi);
    };
    st.f.v = (float)cnt;
    split(cnt > 0 ? dn / (double)cnt : 1.0, st.f.s1h, st.f.s1l);
    split(v0 > 0 ? dn / (double)v0 : 1.0, st.f.s0h, st.f.s0l);
    split(cnt > 0 ? 1.0 / (double)cnt : 1.0, st.f.t1h, st.f.t1l);
    split(v0 > 0 ? 1.0 / (double)v0 : 1.0, st.f.t0h, st.f.t0l);
    st.f.pad[0] = st.f.pad[1] = st.f.pad[2] = 0.f;
    colstat[c] = st;
    if (blkrange) {
        // per-128-column (min, max) of the real columns: one atomic pair per
        // warp (its 32 columns lie in one block) instead of one per column
        int lo = real ? (int)cnt : 0x7FFFFFFF, hi = real ? (int)cnt : -1;
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, hi);
        if ((threadIdx.x & 31) == 0 && hi >= 0) {
            atomicMin(&blkrange[c / 128].x, lo);
            atomicMax(&blkrange[c / 128].y, hi);
        }
    }
}

}  // namespace mib200
