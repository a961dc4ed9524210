// hmma_bench.cu -- legacy mma.sync.m16n8k16 (f16 x f16 -> f32) throughput per SM on
// sm_100a: W warps per CTA (one CTA per SM), each with 4 independent accumulator
// chains; reports FLOP per SM-cycle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/hmma_bench tools/hmma_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(int iters, float* out, unsigned long long* cyc) {
    uint32_t a0 = threadIdx.x * 0x00010001u, a1 = a0 ^ 0x3c003c00u, a2 = a0 + 1u, a3 = a1 + 3u;
    uint32_t b0 = a0 ^ 0x12341234u, b1 = a1 ^ 0x4321u;
    float c[4][4] = {};
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
    for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    float* d;
    unsigned long long* c;
    cudaMalloc(&d, 148 * 1024 * 4);
    cudaMalloc(&c, 8);
    const int iters = 2000;
    for (int w : {1, 2, 4, 8, 16}) {
        k<<<148, 32 * w>>>(iters, d, c);
        cudaDeviceSynchronize();
        unsigned long long h;
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        const double flop = 4.0 * iters * w * 4096.0;  // per SM
        printf("warps %2d: %.0f FLOP/SM-cycle (%.1f cycles per mma per warp)\n", w, flop / h, (double)h / (4.0 * iters));
    }
    return 0;
}
