// Pure HBM write bandwidth with hand-written store kernels (16-byte and
// 32-byte stores, default and streaming cache hints, grid sizes), against
// cudaMemset: is ~3.9 TB/s the write ceiling the unpack kernel is held to?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o write_bw write_bw.cu && ./write_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int W, bool CS>
__global__ void wr(uint4* p, size_t n16) {
    const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t nthr = (size_t)gridDim.x * blockDim.x;
    const uint4 v = make_uint4(tid, 1, 2, 3);
    if (W == 16) {
        for (size_t i = tid; i < n16; i += nthr) {
            if (CS) __stcs(p + i, v); else p[i] = v;
        }
    } else {
        const size_t n32 = n16 / 2;
        for (size_t i = tid; i < n32; i += nthr) {
            uint4* q = p + 2 * i;
            if (CS)
                asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(q), "r"(v.x), "r"(v.y),
                             "r"(v.z), "r"(v.w), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
            else
                asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(q), "r"(v.x), "r"(v.y),
                             "r"(v.z), "r"(v.w), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
        }
    }
}

int main() {
    const size_t bytes = 2ull << 30;
    uint4* p;
    cudaMalloc(&p, bytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, auto launch) {
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(a);
        for (int i = 0; i < 10; ++i) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 10;
        printf("%-40s %.3f ms  %.0f GB/s\n", name, ms, bytes / ms / 1e6);
    };
    run("cudaMemset", [&] { cudaMemsetAsync(p, 0, bytes); });
    for (int blocks_per_sm : {2, 4, 8, 16}) {
        for (int t : {256, 512}) {
            char nm[64];
            const int g = sms * blocks_per_sm;
            snprintf(nm, sizeof nm, "st16    %3d x %d", g, t);
            run(nm, [&] { wr<16, false><<<g, t>>>(p, bytes / 16); });
            snprintf(nm, sizeof nm, "st16.cs %3d x %d", g, t);
            run(nm, [&] { wr<16, true><<<g, t>>>(p, bytes / 16); });
            snprintf(nm, sizeof nm, "st32    %3d x %d", g, t);
            run(nm, [&] { wr<32, false><<<g, t>>>(p, bytes / 16); });
            snprintf(nm, sizeof nm, "st32.cs %3d x %d", g, t);
            run(nm, [&] { wr<32, true><<<g, t>>>(p, bytes / 16); });
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
