// Device -> pinned host bandwidth through SM stores into mapped host memory
// (zero-copy), full rows and strided column strips, against cudaMemcpy2DAsync:
// can a copy kernel beat the copy engines' ~52 GB/s on 2-D regions?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o zc_d2h zc_d2h.cu && ./zc_d2h
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void copy2d(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t pitch16, size_t width16,
                       size_t rows) {
    const size_t n = width16 * rows;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const size_t r = i / width16, c = i - r * width16;
        const uint4 v = __ldcs(src + r * pitch16 + c);
        __stcs(dst + r * pitch16 + c, v);
    }
}

int main() {
    const size_t m = 10000, pitch = m * 8;  // float64 rows of a 10000 x 10000 matrix
    const size_t bytes = m * pitch;
    void *d, *h, *hd;
    cudaMalloc(&d, bytes);
    cudaMemset(d, 1, bytes);
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
    cudaHostGetDevicePointer(&hd, h, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (size_t wcols : {10000, 2500}) {
        const size_t w = wcols * 8;
        for (int grid : {16, 32, 64, 148, 296}) {
            for (int it = 0; it < 2; ++it)
                copy2d<<<grid, 512>>>((const uint4*)d, (uint4*)hd, pitch / 16, w / 16, m);
            cudaEventRecord(a);
            copy2d<<<grid, 512>>>((const uint4*)d, (uint4*)hd, pitch / 16, w / 16, m);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("kernel %3d x 512, %zu rows x %zu B: %.2f ms = %.1f GB/s\n", grid, m, w, ms, m * w / ms / 1e6);
        }
        cudaEventRecord(a);
        cudaMemcpy2DAsync(h, pitch, d, pitch, w, m, cudaMemcpyDeviceToHost, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("cudaMemcpy2DAsync  %zu rows x %zu B: %.2f ms = %.1f GB/s\n", m, w, ms, m * w / ms / 1e6);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
