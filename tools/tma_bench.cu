// tma_bench.cu -- how fast can one SM pull a stream of ~4 KB records into
// shared memory?  Compares cp.async.bulk from one producer lane, from every
// warp, cp.async (LDGSTS) by all lanes, and plain LDG.128 into registers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tma_bench tools/tma_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(sa(b)),
                 "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(d)),
                 "l"(s), "r"(n), "r"(sa(b)) : "memory");
}

// mode 0: one producer lane (warp NW) feeds NW consumer warps through a ring of S slots
__global__ void k_producer(const uint8_t* src, size_t per_cta, uint32_t rec, int S, int NW, unsigned* sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t full[64], empty[64];
    __shared__ unsigned tick;
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        tick = 0;
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const uint8_t* base = src + blockIdx.x * per_cta;
    uint32_t n = per_cta / rec;
    if (warp == NW) {
        if (lane == 0)
            for (uint32_t t = 0; t < n; ++t) {
                uint32_t s = t % S;
                if (t >= (uint32_t)S) wait(&empty[s], ((t / S) - 1) & 1);
                expect_tx(&full[s], rec);
                bulk(sm + (size_t)s * rec, base + (size_t)t * rec, rec, &full[s]);
            }
        return;
    }
    unsigned acc = 0;
    for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(&tick, 1);
        t = __shfl_sync(~0u, t, 0);
        if (t >= n) break;
        uint32_t s = t % S;
        wait(&full[s], (t / S) & 1);
        acc += sm[(size_t)s * rec + lane * 4];
        __syncwarp();
        if (lane == 0) arrive(&empty[s]);
    }
    if (acc == 0xdeadbeef) sink[0] = acc;
}

// mode 1: every warp issues its own records into its own ring of S slots
__global__ void k_perwarp(const uint8_t* src, size_t per_cta, uint32_t rec, int S, int NW, unsigned* sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t full[32][8];
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        for (int i = 0; i < S; ++i) mbar_init(&full[warp][i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    uint8_t* ring = sm + (size_t)warp * S * rec;
    const uint8_t* base = src + blockIdx.x * per_cta;
    uint32_t n = per_cta / rec;
    unsigned acc = 0;
    uint32_t t = warp, k = 0;
    if (lane == 0)
        for (int s = 0; s < S && warp + s * NW < (int)n; ++s) {
            expect_tx(&full[warp][s], rec);
            bulk(ring + s * rec, base + (size_t)(warp + s * NW) * rec, rec, &full[warp][s]);
        }
    for (; t < n; t += NW, ++k) {
        uint32_t s = k % S;
        wait(&full[warp][s], (k / S) & 1);
        acc += ring[s * rec + lane * 4];
        __syncwarp();
        uint32_t tn = t + S * NW;
        if (lane == 0 && tn < n) {
            expect_tx(&full[warp][s], rec);
            bulk(ring + s * rec, base + (size_t)tn * rec, rec, &full[warp][s]);
        }
    }
    if (acc == 0xdeadbeef) sink[0] = acc;
}

// mode 2: plain LDG.128 by all lanes, records interleaved over warps, 4 in flight per lane
__global__ void k_ldg(const uint8_t* src, size_t per_cta, uint32_t rec, int S, int NW, unsigned* sink) {
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint4* base = reinterpret_cast<const uint4*>(src + blockIdx.x * per_cta);
    size_t n16 = per_cta / 16;
    unsigned acc = 0;
    for (size_t i = (size_t)warp * 32 + lane; i < n16; i += (size_t)NW * 32 * 4) {
        uint4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            size_t ii = i + (size_t)j * NW * 32;
            v[j] = ii < n16 ? __ldg(base + ii) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) acc += v[j].x ^ v[j].w;
    }
    if (acc == 0xdeadbeef) sink[0] = acc;
}

int main(int argc, char** argv) {
    const int only = argc > 1 ? atoi(argv[1]) : -1;
    int idx = -1;
    const size_t total = 400ull << 20;
    uint8_t* d;
    unsigned* sink;
    cudaMalloc(&d, total + (1 << 20));
    cudaMalloc(&sink, 4);
    cudaMemset(d, 1, total);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, auto kern, uint32_t rec, int S, int NW, size_t smem, int threads) {
        ++idx;
        if (only >= 0 && idx != only) return;
        size_t per = (total / sms) / rec * rec;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        for (int i = 0; i < 3; ++i) kern<<<sms, threads, smem>>>(d, per, rec, S, NW, sink);
        cudaEventRecord(a);
        for (int i = 0; i < 10; ++i) kern<<<sms, threads, smem>>>(d, per, rec, S, NW, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        cudaError_t e = cudaGetLastError();
        printf("%-12s rec %5u S %2d NW %2d : %7.1f GB/s %s\n", name, rec, S, NW, per * sms * 10 / (ms * 1e-3) / 1e9,
               e ? cudaGetErrorString(e) : "");
    };
    for (uint32_t rec : {2048u, 4096u, 8192u})
        for (int S : {16, 32})
            if ((size_t)S * rec <= 190 * 1024) run("producer", k_producer, rec, S, 15, (size_t)S * rec, 16 * 32);
    for (uint32_t rec : {2048u, 4096u, 8192u})
        for (int S : {2, 3, 4})
            if ((size_t)S * rec * 16 <= 190 * 1024) run("perwarp", k_perwarp, rec, S, 16, (size_t)S * rec * 16, 16 * 32);
    run("ldg", k_ldg, 4096, 0, 16, 0, 16 * 32);
    run("ldg", k_ldg, 4096, 0, 32, 0, 32 * 32);
    return 0;
}
