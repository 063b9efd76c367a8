// Microbenchmark: per-SM throughput of DFMA / DADD / FFMA / IMAD on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int OP>
__global__ void k(T* out, int iters, T a, T b) {
    T x0 = a + threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (OP == 0) {  // fma
                x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
                x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
            } else {        // add
                x0 = x0 + b; x1 = x1 + b; x2 = x2 + b; x3 = x3 + b;
                x4 = x4 + b; x5 = x5 + b; x6 = x6 + b; x7 = x7 + b;
            }
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

template <typename T, int OP>
void run(const char* name, int threads) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    T* out;
    cudaMalloc(&out, sizeof(T) * sms * 4 * threads);
    const int iters = 4096;
    k<T, OP><<<sms * 4, threads>>>(out, 16, (T)1.0000001, (T)0.5);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<T, OP><<<sms * 4, threads>>>(out, iters, (T)1.0000001, (T)0.5);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)sms * 4 * threads * iters * 32;  // lane-ops
    double per_sm_clk = ops / (ms * 1e-3) / sms / (clk * 1e3);
    printf("%-6s threads/blk %4d: %.3f ms, %.1f lane-ops/clk/SM (at %d MHz boost), %.2f Tops/s\n", name, threads, ms,
           per_sm_clk, clk / 1000, ops / (ms * 1e-3) / 1e12);
    cudaFree(out);
}

int main() {
    for (int t : {128, 256, 512}) {
        run<double, 0>("DFMA", t);
        run<double, 1>("DADD", t);
        run<float, 0>("FFMA", t);
        run<int, 0>("IMAD", t);
    }
    return 0;
}
