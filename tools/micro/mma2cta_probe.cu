// Peak of the 2-SM MMA (cta_group::2, M=256, N=256) on smem-resident
// operands: kind::i8 (K=32) vs kind::mxf4 (K=64, unit scales in TMEM), MACs
// per clock per SM over all 74 SM pairs.  Operand contents are irrelevant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2411_19702_b200/csrc -o mma2cta_probe mma2cta_probe.cu
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace mib200;

template <bool FP4>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe(long long* cycles, int reps) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x / 32;
    const uint32_t rank = cluster_ctarank();
    for (int i = threadIdx.x; i < 4 * 2 * 16384 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x22222222u * (i & 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbarrier_init(); }
    if (warp == 0) tmem_alloc<2>(smem_u32(&tslot), 512);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (FP4) {
        const uint32_t one[16] = {0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu,
                                  0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu,
                                  0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu};
        tmem_st_32x32b_x16(tmem + ((uint32_t)(warp * 32) << 16) + 496, one);
        tmem_st_wait();
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (rank == 0 && threadIdx.x == 0) {
        const uint32_t idesc = FP4 ? umma_idesc_mxf4(256, 256) : umma_idesc_i8(256, 256);
        long long t0 = clock64();
        for (int rep = 0; rep < reps; ++rep) {
            for (int kb = 0; kb < 4; ++kb) {
                const uint64_t ad = umma_desc_sw128_kmajor(smem_u32(smem + kb * 32768));
                const uint64_t bd = umma_desc_sw128_kmajor(smem_u32(smem + kb * 32768 + 16384));
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    if (FP4) umma_mxf4<2>(tmem, ad + 2u * s, bd + 2u * s, idesc, tmem + 496, tmem + 496, 1u);
                    else umma_i8<2>(tmem, ad + 2u * s, bd + 2u * s, idesc, 1u);
                }
            }
        }
        umma_commit<2>(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), 0);
        cycles[blockIdx.x / 2] = clock64() - t0;
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 0) tmem_dealloc<2>(tmem, 512);
}

int main() {
    long long* dc;
    cudaMalloc(&dc, 74 * 8);
    const size_t smem = 4 * 32768 + 1024;
    for (int fp4 = 0; fp4 < 2; ++fp4) {
        auto k = fp4 ? probe<true> : probe<false>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int reps = 4000;
        k<<<148, 128, smem>>>(dc, reps);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; }
        std::vector<long long> c(74);
        cudaMemcpy(c.data(), dc, 74 * 8, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (auto x : c) mx = x > mx ? x : mx;
        const double macs_pair = (double)reps * 16 * 256 * 256 * (fp4 ? 64 : 32);
        printf("%s cta_group::2 M256 N256: %.0f MACs/clk/SM\n", fp4 ? "mxf4" : "i8", macs_pair / mx / 2);
    }
    return 0;
}
