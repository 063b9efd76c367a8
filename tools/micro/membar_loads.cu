// Does fence.proxy.async.shared::cta (SASS: MEMBAR.ALL.CTA + FENCE.VIEW.ASYNC.S)
// wait for the thread's outstanding global loads?  One warp issues 8 loads of
// cold lines, then the fence, then reads the clock; the loads' data are used
// only afterwards.  Compared with the same without loads in flight.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(const unsigned long long* __restrict__ g, long long* out, int mode) {
    __shared__ unsigned int s[64];
    const int lane = threadIdx.x;
    unsigned long long v[8];
    long long t0 = clock64();
    if (mode >= 1) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __ldcg(g + (size_t)i * (1 << 20) + lane * 32);  // 8 MB apart: DRAM
    }
    s[lane] = lane;
    long long t1 = clock64();
    if (mode == 2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    long long t2 = clock64();
    unsigned long long acc = 0;
    if (mode >= 1) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc += v[i];
    }
    long long t3 = clock64();
    if (lane == 0) {
        out[0] = t1 - t0;
        out[1] = t2 - t1;
        out[2] = t3 - t2;
        out[3] = (long long)acc + s[3];
    }
}

int main() {
    unsigned long long* g;
    long long* o;
    cudaMalloc(&g, (size_t)8 << 23);
    cudaMemset(g, 1, (size_t)8 << 23);
    cudaMalloc(&o, 64);
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            // evict: touch another big buffer so the lines are cold
            k<<<1, 32>>>(g, o, mode);
            long long h[4];
            cudaMemcpy(h, o, 32, cudaMemcpyDeviceToHost);
            if (rep == 2)
                printf("mode %d (%s): issue %lld, fence %lld, use %lld cycles\n", mode,
                       mode == 0 ? "no loads" : mode == 1 ? "loads, no fence" : "loads + fence", h[0], h[1], h[2]);
        }
    }
    return 0;
}
