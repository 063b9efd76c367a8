// Probe: can tcgen05.mma.kind::mxf4 (e2m1 operands, E8M0 block scales all
// 1.0) compute exact 0/1 Gram counts, and how fast is it against kind::i8?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2411_19702_b200/csrc -o mxf4_probe mxf4_probe.cu
//
// Part 1 (one CTA): A = 128 x K bits, B = 256 x K bits staged in shared memory
// in the SW128 K-major layout (int8: one byte per bit; e2m1: one nibble per
// bit, 1.0 = 0b0010), D = A B^T in TMEM, read back and compared with popcount.
// Part 2 (148 CTAs): clock64 over a long stream of MMAs on resident shared
// memory: MACs per clock per SM for kind::i8 (K=32) and kind::mxf4 (K=64).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace mib200;

constexpr int M = 128, N = 256, KB = 4;  // 4 k-blocks of 128-byte rows

__host__ __device__ constexpr uint32_t idesc_mxf4(int m, int n) {
    return (1u << 7) | (1u << 10)                 // A, B: E2M1 (MXF4 format)
           | (0u << 15) | (0u << 16)              // K-major
           | (static_cast<uint32_t>(n >> 3) << 17)
           | (1u << 23)                           // scale format E8M0
           | (static_cast<uint32_t>(m >> 4) << 24);
}

__device__ __forceinline__ void mma_mxf4(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sfa,
                                         uint32_t sfb, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb)
        : "memory");
}

__device__ __forceinline__ void tmem_st_x32(uint32_t taddr, uint32_t v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
        "%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(taddr),
        "r"(v)
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// byte offset of (row r, byte kbyte in [0,128)) inside one SW128 K-major k-block of `rows` rows
__host__ __device__ inline int sw128(int r, int kbyte) {
    return (r / 8) * 1024 + (r % 8) * 128 + (((kbyte / 16) ^ (r % 8)) * 16) + (kbyte % 16);
}

template <bool FP4>
__global__ void __launch_bounds__(128, 1) gram_probe(const uint8_t* abits, const uint8_t* bbits, float* out_f,
                                                      int* out_i, long long* cycles, int reps, int sfw) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int K = FP4 ? KB * 256 : KB * 128;  // elements per row
    const int warp = threadIdx.x / 32;
    uint8_t* sA = smem;                        // KB blocks of M x 128 B
    uint8_t* sB = smem + KB * M * 128;         // KB blocks of N x 128 B
    // stage operands
    for (int idx = threadIdx.x; idx < KB * (M + N) * 128; idx += blockDim.x) smem[idx] = 0;
    __syncthreads();
    if (abits) {
        for (int idx = threadIdx.x; idx < M * K; idx += blockDim.x) {
            const int r = idx / K, k = idx % K;
            if (!abits[idx]) continue;
            const int kb = FP4 ? k / 256 : k / 128, kin = FP4 ? k % 256 : k % 128;
            uint8_t* base = sA + kb * M * 128;
            if (FP4) atomicOr((unsigned*)(base + (sw128(r, kin / 2) & ~3)), 0x2u << (((sw128(r, kin / 2) & 3) * 8) + 4 * (kin & 1)));
            else base[sw128(r, kin)] = 1;
        }
        for (int idx = threadIdx.x; idx < N * K; idx += blockDim.x) {
            const int r = idx / K, k = idx % K;
            if (!bbits[idx]) continue;
            const int kb = FP4 ? k / 256 : k / 128, kin = FP4 ? k % 256 : k % 128;
            uint8_t* base = sB + kb * N * 128;
            if (FP4) atomicOr((unsigned*)(base + (sw128(r, kin / 2) & ~3)), 0x2u << (((sw128(r, kin / 2) & 3) * 8) + 4 * (kin & 1)));
            else base[sw128(r, kin)] = 1;
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbarrier_init(); }
    if (warp == 0) tmem_alloc<1>(smem_u32(&tslot), 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    // scale factors: columns 256..511 of every lane = 0x7F (E8M0 1.0)
    if (FP4) {
        for (int c = 256; c < 512; c += 32) tmem_st_x32(tmem + ((uint32_t)(warp * 32) << 16) + c, 0x80808080u);
        // sfw columns of 1.0 at SFA (256) and SFB (384), 2.0 elsewhere: exact results <=> the MMA reads
        // no more than sfw columns of scales
        for (int c = 0; c < sfw; ++c) {
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + ((uint32_t)(warp * 32) << 16) + 256 + c), "r"(0x7F7F7F7Fu) : "memory");
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + ((uint32_t)(warp * 32) << 16) + 384 + c), "r"(0x7F7F7F7Fu) : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t idesc = FP4 ? idesc_mxf4(M, N) : umma_idesc_i8(M, N);
        const uint32_t sfa = tmem + 256, sfb = tmem + 384;
        long long t0 = clock64();
        for (int rep = 0; rep < reps; ++rep) {
            for (int kb = 0; kb < KB; ++kb) {
                const uint64_t ad = umma_desc_sw128_kmajor(smem_u32(sA + kb * M * 128));
                const uint64_t bd = umma_desc_sw128_kmajor(smem_u32(sB + kb * N * 128));
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    const uint32_t acc = (rep | kb | s) != 0;
                    if (FP4) mma_mxf4(tmem, ad + 2u * s, bd + 2u * s, idesc, sfa, sfb, acc);
                    else umma_i8<1>(tmem, ad + 2u * s, bd + 2u * s, idesc, acc);
                }
            }
        }
        umma_commit<1>(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), 0);
        long long t1 = clock64();
        if (cycles) cycles[blockIdx.x] = t1 - t0;
    }
    __syncthreads();
    tc_fence_after();
    if (out_f && blockIdx.x == 0) {
        // D: lane = row (32 per warp), column = B row
        const int row = warp * 32 + (threadIdx.x & 31);
        for (int c = 0; c < N; c += 16) {
            uint32_t r[16];
            tmem_ld_32x32b_x16(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
            tmem_ld_wait(r);
            for (int k = 0; k < 16; ++k) {
                if (FP4) out_f[row * N + c + k] = __uint_as_float(r[k]);
                else out_i[row * N + c + k] = (int)r[k];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<1>(tmem, 512);
}

int main() {
    const size_t smem = KB * (M + N) * 128 + 1024;
    for (int fp4 = 0; fp4 < 2; ++fp4) {
        const int K = fp4 ? KB * 256 : KB * 128;
        std::vector<uint8_t> a(M * K), b(N * K);
        srand(1 + fp4);
        for (auto& x : a) x = (rand() % 100) < 40;
        for (auto& x : b) x = (rand() % 100) < 55;
        uint8_t *da, *db;
        float* df;
        int* di;
        long long* dc;
        cudaMalloc(&da, a.size()); cudaMalloc(&db, b.size());
        cudaMalloc(&df, M * N * 4); cudaMalloc(&di, M * N * 4); cudaMalloc(&dc, 148 * 8);
        cudaMemcpy(da, a.data(), a.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(db, b.data(), b.size(), cudaMemcpyHostToDevice);
        auto kern = fp4 ? gram_probe<true> : gram_probe<false>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int sfw = 1; fp4 && sfw <= 64; sfw *= 2) {
            kern<<<1, 128, smem>>>(da, db, df, di, dc, 1, sfw);
            cudaDeviceSynchronize();
            std::vector<float> t(M * N);
            cudaMemcpy(t.data(), df, M * N * 4, cudaMemcpyDeviceToHost);
            long bad = 0;
            for (int i = 0; i < M; ++i)
                for (int j = 0; j < N; ++j) {
                    int ref = 0;
                    for (int k = 0; k < K; ++k) ref += a[i * K + k] & b[j * K + k];
                    bad += t[i * N + j] != (float)ref;
                }
            printf("  mxf4 with %d scale column(s) of 1.0 at SFA and SFB: %ld mismatches\n", sfw, bad);
        }
        kern<<<1, 128, smem>>>(da, db, df, di, dc, 1, 128);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s: %s\n", fp4 ? "mxf4" : "i8", cudaGetErrorString(e)); return 1; }
        std::vector<float> of(M * N);
        std::vector<int> oi(M * N);
        cudaMemcpy(of.data(), df, M * N * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(oi.data(), di, M * N * 4, cudaMemcpyDeviceToHost);
        long bad = 0;
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < N; ++j) {
                int ref = 0;
                for (int k = 0; k < K; ++k) ref += a[i * K + k] & b[j * K + k];
                const double got = fp4 ? (double)of[i * N + j] : (double)oi[i * N + j];
                if (got != (double)ref) {
                    if (bad < 5) printf("  mismatch (%d,%d): got %.1f want %d\n", i, j, got, ref);
                    ++bad;
                }
            }
        printf("%s correctness: K=%d, %ld mismatches of %d\n", fp4 ? "mxf4" : "i8", K, bad, M * N);
        // throughput: all SMs, garbage smem (abits = nullptr skips staging)
        const int reps = 2000;
        kern<<<148, 128, smem>>>(nullptr, nullptr, nullptr, nullptr, dc, reps, 128);
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("throughput run: %s\n", cudaGetErrorString(e)); return 1; }
        std::vector<long long> cyc(148);
        cudaMemcpy(cyc.data(), dc, 148 * 8, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (auto c : cyc) mx = c > mx ? c : mx;
        const double macs = (double)reps * KB * 4 * M * N * (fp4 ? 64 : 32);
        printf("%s throughput: %.0f MACs/clk/SM (max cycles %lld over 148 SMs)\n", fp4 ? "mxf4" : "i8", macs / mx, mx);
        cudaFree(da); cudaFree(db); cudaFree(df); cudaFree(di); cudaFree(dc);
    }
    return 0;
}
