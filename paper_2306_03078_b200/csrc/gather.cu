// gather.cu -- the GATHER = true instantiations of gemv_cta (the band kernel of
// the row-sharded path with the y all-gather fused in; see gemv_cta.cuh and
// spqr_matvec_gather in capi.cu).  A separate translation unit so the build
// compiles them in parallel with capi.cu.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace spqr_dev {
namespace {
template <int BW, int BSZ, bool XLO, bool SHX, int NC>
cudaError_t launch_gather_t(const CtaParams& p, std::uint32_t grid, std::uint32_t smem, std::uint32_t smem_limit,
                            cudaStream_t st) {
    auto kern = gemv_cta<BW, BSZ, BSZ, XLO ? 1 : 0, NC, SHX, true>;
    static bool attr_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        cudaFuncAttributes fa{};
        cudaError_t e = cudaFuncGetAttributes(&fa, kern);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem_limit - fa.sharedSizeBytes));
        if (e != cudaSuccess) return e;
        attr_set[dev & 63] = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NC * 32);
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

cudaError_t launch_cta_gather(int bw, int bsz, bool xlo, bool shx, const CtaParams& p, std::uint32_t grid,
                              std::uint32_t smem, int nc, std::uint32_t smem_limit, cudaStream_t st) {
#ifndef SPQR_NC
#define SPQR_NC 16
#endif
    if (nc != SPQR_NC) return cudaErrorInvalidConfiguration;
    const int key = bw * 1000 + bsz * 100 + (xlo ? 10 : 0) + (shx ? 1 : 0);
    switch (key) {
#define SPQR_CASE(BW, BSZ)                                                                                       \
    case BW * 1000 + BSZ * 100 + 0: return launch_gather_t<BW, BSZ, false, false, SPQR_NC>(p, grid, smem, smem_limit, st); \
    case BW * 1000 + BSZ * 100 + 1: return launch_gather_t<BW, BSZ, false, true, SPQR_NC>(p, grid, smem, smem_limit, st);  \
    case BW * 1000 + BSZ * 100 + 10: return launch_gather_t<BW, BSZ, true, false, SPQR_NC>(p, grid, smem, smem_limit, st); \
    case BW * 1000 + BSZ * 100 + 11: return launch_gather_t<BW, BSZ, true, true, SPQR_NC>(p, grid, smem, smem_limit, st);
        SPQR_CASE(2, 2) SPQR_CASE(2, 3) SPQR_CASE(2, 4)
        SPQR_CASE(3, 2) SPQR_CASE(3, 3) SPQR_CASE(3, 4)
        SPQR_CASE(4, 2) SPQR_CASE(4, 3) SPQR_CASE(4, 4)
#undef SPQR_CASE
        default: return cudaErrorInvalidConfiguration;
    }
}
}  // namespace spqr_dev
