// Tensor-peak probe (C ABI mi_tensor_peak): the ceiling the fused kernel's
// roofline is quoted against, measured on the box that runs the bench.
//
// Every SM pair issues back-to-back tcgen05.mma.cta_group::2 (M = 256,
// N = 256) on shared-memory-resident operands -- the fused kernel's own
// instruction, kind::mxf4 with unit block scales (K = 64) or kind::i8
// (K = 32) -- with no operand traffic and no epilogue, so the result is the
// instruction's throughput at the clocks the box runs at (power-capped when
// the run is long).  Operand contents are irrelevant to the rate.
#include <cuda_runtime.h>
#include <cstdint>

#include "mi_kernels.h"
#include "ptx.cuh"

namespace mib200 {

namespace {

constexpr int kProbeKb = 4;  // 4 resident 32 KB stages (A half + B half each)

template <bool FP4>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
tensor_peak_kernel(long long* cycles, int reps) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x / 32;
    const uint32_t rank = cluster_ctarank();
    for (int i = threadIdx.x; i < kProbeKb * 2 * 16384 / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(smem)[i] = 0x22222222u * (i & 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
        fence_mbarrier_init();
    }
    if (warp == 0) tmem_alloc<2>(smem_u32(&tslot), 512);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (FP4) {  // E8M0 scales = 1.0 in columns [496, 512), as in the fused kernel
        const uint32_t one[16] = {0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu,
                                  0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu,
                                  0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu};
        tmem_st_32x32b_x16(tmem + ((uint32_t)(warp * 32) << 16) + 496, one);
        tmem_st_wait();
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (rank == 0 && warp == 1) {
        const uint32_t idesc = FP4 ? umma_idesc_mxf4(256, 256) : umma_idesc_i8(256, 256);
        const uint64_t ad0 = umma_desc_sw128_kmajor(smem_u32(smem));
        const uint64_t bd0 = umma_desc_sw128_kmajor(smem_u32(smem + 16384));
        const long long t0 = clock64();
        for (int rep = 0; rep < reps; ++rep) {
            for (int kb = 0; kb < kProbeKb; ++kb) {
                const uint64_t off = (uint64_t)(kb * (32768 >> 4));
                if (elect_one()) {
#pragma unroll
                    for (int s = 0; s < 4; ++s) {
                        if (FP4) umma_mxf4<2>(tmem, ad0 + off + 2u * s, bd0 + off + 2u * s, idesc, tmem + 496, tmem + 496, 1u);
                        else umma_i8<2>(tmem, ad0 + off + 2u * s, bd0 + off + 2u * s, idesc, 1u);
                    }
                }
                __syncwarp();
            }
        }
        if (elect_one()) umma_commit<2>(smem_u32(&bar));
        __syncwarp();
        mbar_wait(smem_u32(&bar), 0);
        if (threadIdx.x == 32) cycles[blockIdx.x / 2] = clock64() - t0;
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 0) tmem_dealloc<2>(tmem, 512);
}

}  // namespace

cudaError_t launch_tensor_peak(bool fp4, int reps, int num_sms, long long* d_cycles, cudaStream_t stream) {
    const size_t smem = (size_t)kProbeKb * 32768 + 1024;
    auto k = fp4 ? tensor_peak_kernel<true> : tensor_peak_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<(unsigned)(num_sms / 2 * 2), 128, smem, stream>>>(d_cycles, reps);
    return cudaGetLastError();
}

// MACs one probe launch performs per SM pair: reps x kProbeKb x 4 MMAs of 256 x 256 x K.
double tensor_peak_macs_per_pair(bool fp4, int reps) {
    return (double)reps * kProbeKb * 4 * 256.0 * 256.0 * (fp4 ? 64.0 : 32.0);
}

}  // namespace mib200
