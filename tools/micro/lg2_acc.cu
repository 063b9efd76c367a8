// Accuracy of MUFU lg2.approx.f32 (and of the rcp/compensated ratio used by
// the float32 MI epilogue) against a double-precision log2, over every float
// in [2^-4, 2^4) -- the inputs the epilogue feeds it are ratios c N / (a b)
// of counts, so the absolute error of log2 near 1 is what matters.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lg2_acc lg2_acc.cu
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ float lg2_approx(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ unsigned long long g_worst_bits;   // max |err| as ordered double bits
__device__ unsigned int g_worst_x;

__global__ void sweep(unsigned int first, unsigned int count) {
    unsigned long long worst = 0;
    unsigned int wx = 0;
    for (unsigned int k = blockIdx.x * blockDim.x + threadIdx.x; k < count; k += gridDim.x * blockDim.x) {
        const unsigned int bits = first + k;
        const float x = __uint_as_float(bits);
        const double err = fabs((double)lg2_approx(x) - log2((double)x));
        const unsigned long long eb = (unsigned long long)__double_as_longlong(err);
        if (eb > worst) { worst = eb; wx = bits; }
    }
    unsigned long long prev = atomicMax(&g_worst_bits, worst);
    if (worst > prev) g_worst_x = wx;
}

int main() {
    const unsigned int lo = 0x3D800000u;  // 2^-4
    const unsigned int hi = 0x41800000u;  // 2^4
    unsigned long long zero = 0;
    cudaMemcpyToSymbol(g_worst_bits, &zero, 8);
    sweep<<<148 * 8, 256>>>(lo, hi - lo);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error: %s\n", cudaGetErrorString(e)); return 1; }
    unsigned long long wb;
    unsigned int wx;
    cudaMemcpyFromSymbol(&wb, g_worst_bits, 8);
    cudaMemcpyFromSymbol(&wx, g_worst_x, 4);
    double w;
    memcpy(&w, &wb, 8);
    float x;
    memcpy(&x, &wx, 4);
    printf("lg2.approx.ftz.f32 over [2^-4, 2^4): max |err| = %.3e (= 2^%.2f) at x = %.9g\n", w, log2(w), x);
    return 0;
}
