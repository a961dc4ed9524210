// gemm_ex.cu -- the gemm_ex instantiations (exact-code batched decode on the
// tcgen05 tensor cores, gemm_ex.cuh).  A separate translation unit so the
// build compiles them in parallel with capi.cu.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace spqr_dev {
namespace {
template <int BW, int BS, int N>
cudaError_t launch_ex_t(const ExParams& p, std::uint32_t smem, std::uint32_t smem_limit, cudaStream_t st) {
    auto kern = gemm_ex<BW, BS, N>;
    static bool attr_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        cudaFuncAttributes fa{};
        cudaError_t e = cudaFuncGetAttributes(&fa, kern);
        if (e != cudaSuccess) return e;
        if (fa.sharedSizeBytes > kExStaticMax) return cudaErrorInvalidConfiguration;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem_limit - kExStaticMax));
        if (e != cudaSuccess) return e;
        attr_set[dev & 63] = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.nv);
    cfg.blockDim = dim3(kExThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
}
}  // namespace

cudaError_t launch_gemm_ex(int bw, int bs, int n, const ExParams& p, std::uint32_t smem, std::uint32_t smem_limit,
                           cudaStream_t st) {
    const int key = bw * 100 + bs * 10 + (n == 16 ? 0 : (n == 32 ? 1 : 2));
    switch (key) {
#define SPQR_CASE(BW, BS)                                                                 \
    case BW * 100 + BS * 10 + 0: return launch_ex_t<BW, BS, 16>(p, smem, smem_limit, st); \
    case BW * 100 + BS * 10 + 1: return launch_ex_t<BW, BS, 32>(p, smem, smem_limit, st); \
    case BW * 100 + BS * 10 + 2: return launch_ex_t<BW, BS, 64>(p, smem, smem_limit, st);
        SPQR_CASE(2, 2) SPQR_CASE(2, 3) SPQR_CASE(2, 4)
        SPQR_CASE(3, 2) SPQR_CASE(3, 3) SPQR_CASE(3, 4)
        SPQR_CASE(4, 2) SPQR_CASE(4, 3) SPQR_CASE(4, 4)
#undef SPQR_CASE
        default: return cudaErrorInvalidConfiguration;
    }
}
namespace {
template <int BW, int BS, int MT>
cudaError_t launch_bm_t(const ExParams& p, std::uint32_t smem, std::uint32_t smem_limit, cudaStream_t st) {
    auto kern = gemm_bm<BW, BS, MT>;
    static bool attr_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        cudaFuncAttributes fa{};
        cudaError_t e = cudaFuncGetAttributes(&fa, kern);
        if (e != cudaSuccess) return e;
        if (fa.sharedSizeBytes > kExStaticMax) return cudaErrorInvalidConfiguration;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem_limit - kExStaticMax));
        if (e != cudaSuccess) return e;
        attr_set[dev & 63] = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.nv);
    cfg.blockDim = dim3(kBmWarps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
}
}  // namespace

cudaError_t launch_gemm_bm(int bw, int bs, int mt, const ExParams& p, std::uint32_t smem, std::uint32_t smem_limit,
                           cudaStream_t st) {
    const int key = bw * 100 + bs * 10 + mt;
    switch (key) {
#define SPQR_CASE(BW, BS)                                                                \
    case BW * 100 + BS * 10 + 1: return launch_bm_t<BW, BS, 1>(p, smem, smem_limit, st); \
    case BW * 100 + BS * 10 + 2: return launch_bm_t<BW, BS, 2>(p, smem, smem_limit, st);
        SPQR_CASE(2, 2) SPQR_CASE(2, 3) SPQR_CASE(2, 4)
        SPQR_CASE(3, 2) SPQR_CASE(3, 3) SPQR_CASE(3, 4)
        SPQR_CASE(4, 2) SPQR_CASE(4, 3) SPQR_CASE(4, 4)
#undef SPQR_CASE
        default: return cudaErrorInvalidConfiguration;
    }
}
}  // namespace spqr_dev

#ifdef SPQR_TIMELINE
// tools-only: this translation unit's copy of the per-warp wait counters
extern "C" int spqr_debug_ex_timeline(unsigned long long* host, size_t count) {
    return cudaMemcpyFromSymbol(host, spqr_dev::g_timeline,
                                8 * (count < 148 * 32 * 8 ? count : 148 * 32 * 8)) == cudaSuccess ? 0 : 1;
}
#endif
