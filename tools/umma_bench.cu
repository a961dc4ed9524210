// umma_bench.cu -- issue cost of small tcgen05.mma (M = 128, K = one 16-column
// f16 block, N = 16 / 32 / 64) from shared memory, no-swizzle K-major core
// matrices (gemm_ex's layout): one thread issues ITERS x 4 MMAs into a
// 3-slot accumulator ring and commits per slot; reports cycles per MMA with
// and without waiting for completion, for f16 and tf32.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/umma_bench tools/umma_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(sa(b)),
                 "r"(ph) : "memory");
}

template <int N, int SWZ, int MODE, int TS = 0, int WARP = 0>
__global__ void k(int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];  // A 16 KB (4 blocks), B 4 x 16N
    __shared__ uint64_t bar[3];
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (16384 + 256 * 128) / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        for (int i = 0; i < 3; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    if (WARP ? threadIdx.x < 32 : threadIdx.x == 0) {
        constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
        constexpr int SBK = 128 / N >= 4 ? 4 : 128 / N;
        const uint32_t a0 = sa(sm), b0 = a0 + 16384;
        const uint64_t da0 = SWZ ? desc(a0, 16, 1024) | (2ull << 61) : desc(a0, 2048, 128);
        const uint64_t db0 = SWZ ? desc(b0, 16, 1024) | (2ull << 61) : desc(b0, 16 * N, 128);
        constexpr uint64_t ainc = SWZ ? 2 : 256, binc = SWZ ? 2 : 2 * N;  // per block, 16-B units
        long long t0 = clock64();
        uint32_t slot = 0, r = 0, ph = 0;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int blk = 0; blk < 4; ++blk) {
                const uint32_t d = MODE == 2 ? tm : tm + r * 128 + (blk % SBK) * N;
                if (WARP)  // the whole warp runs the loop (uniform operands), one elected lane issues
                    asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                                 "r"(tm + 416 + 8 * blk), "l"(db0 + blk * binc), "n"(idesc), "n"(MODE == 2 ? 1 : 0));
                else if (TS)  // A from TMEM columns 416 + 8 blk
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                                 "r"(tm + 416 + 8 * blk), "l"(db0 + blk * binc), "n"(idesc), "n"(MODE == 2 ? 1 : 0));
                else
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
                             "l"(da0 + blk * ainc), "l"(db0 + blk * binc), "n"(idesc), "n"(MODE == 2 ? 1 : 0));
                if (blk % SBK == SBK - 1) {
                    if (MODE == 1 && slot >= 3) wait(&bar[r], ph ^ 1);
                    if (WARP)
                        asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(sa(&bar[r])) : "memory");
                    else
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar[r])) : "memory");
                    ++slot;
                    if (++r == 3) { r = 0; ph ^= 1; }
                }
            }
        }
        long long t1 = clock64();
        for (int q = 0; q < 3; ++q) {
            const int cnt = (int)(slot - q + 2) / 3;
            if (cnt > 0) wait(&bar[q], (cnt - 1) & 1);
        }
        long long t2 = clock64();
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            out[0] = t1 - t0;
            out[1] = t2 - t0;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, int SWZ, int MODE, int TS = 0, int WARP = 0>
void run(unsigned long long* d) {
    const int iters = 400;
    auto kern = k<N, SWZ, MODE, TS, WARP>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    kern<<<148, 128, 16384 + 256 * 128>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("f16 %s%s N=%d %s: issue %.1f cyc/mma, complete %.1f cyc/mma (%s)\n", SWZ ? "sw128" : "plain", TS ? (WARP ? " A-in-TMEM warp" : " A-in-TMEM") : "", N,
           MODE == 2 ? "same-acc " : (MODE ? "ring-wait" : "no-wait  "), (double)h[0] / (4.0 * iters),
           (double)h[1] / (4.0 * iters), cudaGetErrorString(e));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    run<16, 0, 0, 1>(d); run<16, 0, 1, 1>(d); run<16, 0, 2, 1>(d);
    run<16, 0, 0, 1, 1>(d); run<16, 0, 1, 1, 1>(d); run<16, 0, 2, 1, 1>(d);
    run<64, 0, 0, 1, 1>(d); run<64, 0, 1, 1, 1>(d); run<64, 0, 2, 1, 1>(d);
    run<128, 0, 2, 1, 1>(d);
    return 0;
}
