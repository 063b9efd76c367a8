// Does concurrent tcgen05 int8 MMA work slow down FP64 / FP32 / INT math on
// the same SM?  Warp 0 (lane 0) streams tcgen05.mma.kind::i8 (M=128, N=256,
// K=32) over garbage shared memory while warps 1..8 run an ALU loop; we time
// the ALU loop with clock64, with and without the MMA stream.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2411_19702_b200/csrc -o mma_contention mma_contention.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace mib200;

template <int OP>
__device__ __forceinline__ void alu_loop(double* sink, int iters) {
    if (OP == 0) {
        double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, a = 1.0000001, b = 0.5;
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int u = 0; u < 8; ++u) { x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b); }
        }
        sink[threadIdx.x] = x0 + x1 + x2 + x3;
    } else if (OP == 1) {
        float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, a = 1.0000001f, b = 0.5f;
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int u = 0; u < 8; ++u) { x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b); }
        }
        sink[threadIdx.x] = x0 + x1 + x2 + x3;
    } else {
        int x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, a = 3, b = 7;
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int u = 0; u < 8; ++u) { x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b; }
        }
        sink[threadIdx.x] = x0 + x1 + x2 + x3;
    }
}

template <int OP>
__global__ void __launch_bounds__(288, 1) kern(double* sink, long long* times, int iters, int mma_on) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tslot;
    __shared__ uint64_t bar;
    __shared__ volatile int stop;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); stop = 0; fence_mbarrier_init(); }
    if (warp == 0) tmem_alloc<1>(smem_u32(&tslot), 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 0) {
        if (mma_on && threadIdx.x == 0) {
            const uint32_t idesc = umma_idesc_i8(128, 256);
            const uint64_t ad = umma_desc_sw128_kmajor(smem_u32(smem));
            const uint64_t bd = umma_desc_sw128_kmajor(smem_u32(smem) + 16384);
            uint32_t ph = 0;
            long long n = 0;
            while (!stop) {
                for (int k = 0; k < 64; ++k) umma_i8<1>(tmem, ad + 2u * (k & 3), bd + 2u * (k & 3), idesc, 1u);
                umma_commit<1>(smem_u32(&bar));
                mbar_wait(smem_u32(&bar), ph);
                ph ^= 1u;
                ++n;
            }
            times[blockIdx.x * 4 + 2] = n;
        }
    } else {
        const long long t0 = clock64();
        alu_loop<OP>(sink + blockIdx.x * 288, iters);
        const long long t1 = clock64();
        __syncwarp();
        if (threadIdx.x == 32) times[blockIdx.x * 4 + 0] = t1 - t0;
    }
    // the ALU warps signal the MMA warp to stop
    __syncwarp();
    if (threadIdx.x == 32) stop = 1;
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc<1>(tmem, 256);
}

template <int OP>
void run(const char* name, int mma_on, double* sink, long long* times, int sms) {
    const int iters = 20000;
    cudaFuncSetAttribute(kern<OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    kern<OP><<<sms, 288, 65536>>>(sink, times, iters, mma_on);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
    long long h[4];
    cudaMemcpy(h, times, sizeof(h), cudaMemcpyDeviceToHost);
    const double ops = 8.0 * 32 * 4.0 * 8 * iters;  // 8 warps x 32 lanes x (4 chains x 8 unroll) x iters
    printf("%-5s mma=%d: ALU loop %lld cycles -> %.1f lane-ops/clk/SM  (mma batches %lld)\n", name, mma_on, h[0],
           ops / h[0], h[2]);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* sink;
    long long* times;
    cudaMalloc(&sink, sizeof(double) * 288 * sms);
    cudaMalloc(&times, sizeof(long long) * 4 * sms);
    for (int mma = 0; mma < 2; ++mma) {
        run<0>("DFMA", mma, sink, times, sms);
        run<1>("FFMA", mma, sink, times, sms);
        run<2>("IMAD", mma, sink, times, sms);
    }
    return 0;
}
