// capi.cu -- device side of the C ABI: layer handles (validate, transcode,
// upload), matvec / dequantize launches, export, dense comparator.
//
// Replaces (reference, /root/reference/proj/include/spqr):
//   decode + build_tile_plan ... spqr_layer_create   (format.hpp:354, kernel.hpp:54)
//   dequantize_full ............ spqr_dequantize     (kernel.hpp:17-25)
//   matvec ..................... spqr_matvec[_ws|_host] (kernel.hpp:89-128)
//   encode (of the layer) ...... spqr_layer_export_stream (format.hpp:269)
// No CPU fallback: every compute entry point launches sm_100a kernels or fails
// with SPQR_E_CUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "internal.hpp"
#include "kernels.cuh"

using spqr::detail::guard;
namespace T = spqr_tiled;

namespace {

constexpr std::uint32_t kSmemLimit = 232448;  // 227 KB per CTA on sm_100

thread_local int g_launches = 0;

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string("CUDA: ") + what + ": " + cudaGetErrorString(e));
}

template <class T_>
T_* dalloc(std::size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    ck(cudaMalloc(&p, count * sizeof(T_)), "cudaMalloc");
    return static_cast<T_*>(p);
}

struct DevGuard {
    int prev = -1;
    explicit DevGuard(int dev) {
        cudaGetDevice(&prev);
        if (dev >= 0 && dev != prev) ck(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DevGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

}  // namespace

struct spqr_layer {
    int device = 0;
    spqr_layer_info info{};
    std::vector<std::uint8_t> prefix;  // header + permutation (for export)
    spqr::detail::StreamView geo;      // geometry (base -> prefix)
    // raw stream (dequantize + generic matvec)
    std::uint8_t* d_stream = nullptr;
    std::uint32_t* d_order = nullptr;  // solve position -> source column, or null
    // tiled fast path
    bool fast = false;
    bool exact = false;  // batched calls on exact-code kernels only (spqr_layer_set_exact)
    bool stacked = false;  // several streams stacked row-wise (matvec only)
    std::uint8_t* d_cells = nullptr;
    std::uint32_t* d_cell_off = nullptr;
    std::uint32_t* d_usplit = nullptr;  // gemm_bm: per cell, first outlier entry of the second unit | end << 16
    std::uint32_t Gn = 0, Pn = 0, cell_bytes = 0, n_pad = 0;
    // gemv_cta plan, per x mode (0: f16, 1: f32 hi/lo, 2: f16 batch pair:
    // the panel and row-sum sizes differ)
    struct CtaPlan {
        std::uint32_t nvcta = 0, grid = 0, nslot_log2 = 0, slot_bytes = 0, rec_cap = 0;
        std::uint32_t pan_off = 0, part_off = 0, off_off = 0, gd_off = 0, part_cap = 0, smem = 0;
        bool shared_x = false;  // x panels prepared once per CTA (they fit in shared memory)
        std::uint32_t* d_start = nullptr;  // [nvcta+1]
        std::uint32_t* d_first = nullptr;  // [grid][kNC][2] record byte range of warp w's first cell
        std::vector<std::uint32_t> h_start;  // cta_start on the host (the first grid + 1 go by value)
    } cta[3];
    std::uint32_t pn_magic = 0;
    // gemm_tc plan (batch >= 2): ranges of (128-row tile, panel) units
    struct TcPlan {
        std::uint32_t nv = 0, Tn = 0, pslots = 0, slot_bytes = 0;
        int sigma = 0;
        std::uint32_t* d_start = nullptr;  // [nv+1]
        std::uint32_t* d_maps = nullptr;   // gmap [2*Tn] then cmap [2*nv]
    } tcp;
    // gemm_ex plan (exact-code batched decode): shares tcp's ranges and partial
    // slots; ok = every outlier fits binary16 after the 2^p_c column pre-scale
    // (|v| < 512) and the stage buffers fit shared memory
    struct ExPlan {
        bool ok = false;
        std::uint32_t slot_bytes = 0;
    } exp;
    // own workspace
    mutable std::mutex mu;
    mutable void* d_ws = nullptr;        // device-buffer API (spqr_matvec / _stage / _gather)
    mutable std::uint64_t ws_bytes = 0;
    mutable void* d_wsh = nullptr;       // host-buffer API (spqr_matvec_host): baked into hgraph
    mutable std::uint64_t wsh_bytes = 0;
    mutable float* d_xh = nullptr;  // host-API staging
    mutable float* d_yh = nullptr;
    mutable std::size_t xh_cap = 0, yh_cap = 0;
    // spqr_matvec_host: own non-blocking stream, pinned staging (used when the
    // caller's buffers are pageable), and the [H2D x, kernels, D2H y] sequence
    // as one CUDA graph keyed by (batch, host source, host destination)
    mutable cudaStream_t hst = nullptr;
    mutable float* h_x = nullptr;
    mutable float* h_y = nullptr;
    mutable cudaGraphExec_t hgraph = nullptr;
    mutable int hg_batch = 0, hg_launches = 0;
    mutable const void* hg_src = nullptr;
    mutable void* hg_dst = nullptr;
    // completion: signal_host posts *d_seq + 1 to *h_flag; h_seq = last seen
    mutable std::uint32_t* h_flag = nullptr;
    mutable std::uint32_t* d_seq = nullptr;
    mutable std::uint32_t h_seq = 0;
    // page-locked or not, per caller pointer (cudaPointerGetAttributes once)
    mutable const void* pk_ptr[2] = {nullptr, nullptr};
    mutable bool pk_pinned[2] = {false, false};

    ~spqr_layer() {
        if (hgraph) cudaGraphExecDestroy(hgraph);
        if (hst) cudaStreamDestroy(hst);
        if (h_x) cudaFreeHost(h_x);
        if (h_y) cudaFreeHost(h_y);
        if (h_flag) cudaFreeHost(h_flag);
        if (d_seq) cudaFree(d_seq);
        for (void* p : {static_cast<void*>(d_stream), static_cast<void*>(d_order), static_cast<void*>(d_cells),
                        static_cast<void*>(d_cell_off), static_cast<void*>(d_usplit), d_ws, d_wsh,
                        static_cast<void*>(cta[0].d_start), static_cast<void*>(cta[1].d_start),
                        static_cast<void*>(cta[2].d_start), static_cast<void*>(cta[0].d_first),
                        static_cast<void*>(cta[1].d_first), static_cast<void*>(cta[2].d_first),
                        static_cast<void*>(tcp.d_start), static_cast<void*>(tcp.d_maps),
                        static_cast<void*>(d_xh), static_cast<void*>(d_yh)})
            if (p) cudaFree(p);
    }
};

namespace {

spqr_dev::RawGeom raw_geom_of(const spqr::detail::StreamView& v, const std::uint8_t* d_stream,
                              const std::uint32_t* d_order) {
    spqr_dev::RawGeom g{};
    g.s = d_stream;
    g.order = d_order;
    g.rows = v.rows; g.cols = v.cols; g.b1 = v.b1; g.b2 = v.b2;
    g.nblocks = v.nblocks; g.ngroups = v.ngroups;
    g.wb = v.wb; g.sb = v.sb; g.zb = v.zb;
    g.rec_off = v.rec_off; g.col_block_bytes = v.col_block_bytes;
    g.csr_off = v.csr_off; g.ent_off = v.ent_off;
    return g;
}

spqr_dev::RawGeom raw_geom(const spqr_layer* L) {
    const auto& v = L->geo;
    spqr_dev::RawGeom g{};
    g.s = L->d_stream;
    g.order = L->d_order;
    g.rows = v.rows; g.cols = v.cols; g.b1 = v.b1; g.b2 = v.b2;
    g.nblocks = v.nblocks; g.ngroups = v.ngroups;
    g.wb = v.wb; g.sb = v.sb; g.zb = v.zb;
    g.rec_off = v.rec_off; g.col_block_bytes = v.col_block_bytes;
    g.csr_off = v.csr_off; g.ent_off = v.ent_off;
    return g;
}

// Workspace carve-up (bytes, 256-aligned pieces).  The regions the kernels
// count in (xcnt, tc_cnt) must be zero before the first launch; every launch
// leaves them zero again.
struct WsLayout {
    std::uint64_t xpart = 0, xcnt = 0, xp = 0;
    std::uint64_t tc_x = 0, tc_part = 0, tc_cnt = 0, ex_x = 0, ex_scale = 0, total = 0;
};
std::uint64_t al(std::uint64_t v) { return (v + 255) & ~std::uint64_t{255}; }
WsLayout ws_layout(const spqr_layer* L, int batch) {
    WsLayout w;
    const std::uint64_t b = static_cast<std::uint64_t>(std::max(batch, 1));
    std::uint64_t o = 0;
    if (L->fast) {
        // pairs shared by two gemv_cta ranges: partial rows + arrival tickets
        // (two batch columns per boundary for the batch-pair kernel)
        const std::uint64_t nb = std::max({L->cta[0].nvcta, L->cta[1].nvcta, L->cta[2].nvcta}) + 1ull;
        w.xpart = o; o += al(nb * 2 * 2 * 32 * 4);
        w.xcnt = o; o += al(nb * 2 * 4);
        if (batch >= 2) {  // gemm_tc: x tiles for N <= 128, partial tiles, per-warp tile counters
            w.tc_x = o; o += al(static_cast<std::uint64_t>(2 * L->Pn) * 256 * 128);
            w.tc_part = o; o += al(static_cast<std::uint64_t>(L->tcp.pslots) * 128 * 128 * 4);
            w.tc_cnt = o; o += al(static_cast<std::uint64_t>(L->tcp.Tn) * 16 * 4);
            if (L->exact && L->exp.ok) {  // gemm_ex: x tiles of every stage (N <= 64, fp32 x), column scales
                w.ex_x = o; o += al(4ull * L->Pn * std::max(spqr_dev::ex_xbytes(64, true), spqr_dev::ex_xbytes(64, false)));
                w.ex_scale = o; o += al(64 * 4);
            }
        }
    } else {
        w.xp = o; o += al(b * L->info.cols * 4);
    }
    w.total = o;
    return w;
}

// ---- gemv_cta (v14): kNC warps per CTA, one CTA per SM ------------------
#ifndef SPQR_NC
#define SPQR_NC 16
#endif
constexpr int kNC = SPQR_NC;  // 16: 4 warps per SMSP, up to 128 registers each
constexpr std::uint32_t kCtaStaticMax = 10240;  // static smem of gemv_cta (checked at first launch)

template <int BW, int BSZ, int XM, bool SHX>
void launch_cta_t(const spqr_dev::CtaParams& p, std::uint32_t grid, std::uint32_t smem, cudaStream_t st) {
    auto kern = spqr_dev::gemv_cta<BW, BSZ, BSZ, XM, kNC, SHX>;
    static bool attr_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        cudaFuncAttributes fa{};
        ck(cudaFuncGetAttributes(&fa, kern), "cudaFuncGetAttributes(gemv_cta)");
        if (fa.sharedSizeBytes > kCtaStaticMax)
            throw CudaError("gemv_cta: static shared memory exceeds the planned budget");
        ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kSmemLimit - kCtaStaticMax)),
           "cudaFuncSetAttribute(gemv_cta smem)");
        attr_set[dev & 63] = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kNC * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ck(cudaLaunchKernelEx(&cfg, kern, p), "launch gemv_cta");
    ++g_launches;
}

void dispatch_cta(const spqr_dev::CtaParams& p, const spqr_layer* L, int xm, cudaStream_t st) {
    const auto& c = L->cta[xm];
    const int key = L->info.weight_bits * 1000 + L->info.scale_bits * 100 + xm * 10 + (c.shared_x ? 1 : 0);
    switch (key) {
#define SPQR_CASE(BW, BSZ)                                                                           \
    case BW * 1000 + BSZ * 100 + 0: launch_cta_t<BW, BSZ, 0, false>(p, c.grid, c.smem, st); break;  \
    case BW * 1000 + BSZ * 100 + 1: launch_cta_t<BW, BSZ, 0, true>(p, c.grid, c.smem, st); break;   \
    case BW * 1000 + BSZ * 100 + 10: launch_cta_t<BW, BSZ, 1, false>(p, c.grid, c.smem, st); break; \
    case BW * 1000 + BSZ * 100 + 11: launch_cta_t<BW, BSZ, 1, true>(p, c.grid, c.smem, st); break;  \
    case BW * 1000 + BSZ * 100 + 20: launch_cta_t<BW, BSZ, 2, false>(p, c.grid, c.smem, st); break; \
    case BW * 1000 + BSZ * 100 + 21: launch_cta_t<BW, BSZ, 2, true>(p, c.grid, c.smem, st); break;
        SPQR_CASE(2, 2) SPQR_CASE(2, 3) SPQR_CASE(2, 4)
        SPQR_CASE(3, 2) SPQR_CASE(3, 3) SPQR_CASE(3, 4)
        SPQR_CASE(4, 2) SPQR_CASE(4, 3) SPQR_CASE(4, 4)
#undef SPQR_CASE
        default: spqr::fail(spqr::Errc::config_invalid, "no gemv_cta kernel instantiated for this layer");
    }
}


// ---- gemm_tc (batch >= 2): 4 dequant warps + 1 control warp per CTA -------
constexpr std::uint32_t kTcStaticMax = 2048;
constexpr std::uint32_t kTcMaxN = 64;  // batch columns per launch
// below this batch, gemv_cta launches (batch-pair kernels, each weight decoded
// once per two columns) beat the dequant-then-MMA kernel (tools/batch_sweep.py,
// 8192x22016: batch 4 = 2 x 38 us < 84 us; batch 5 = 2 x 38 + 29 us > ~85 us)
constexpr int kTcMinBatch = 5;
std::uint32_t tc_smem(const spqr_layer* L, std::uint32_t N, std::uint32_t na) {
    return na * 128u * 128u * 2u + 3u * 256u * N + 8u * L->tcp.slot_bytes + spqr_dev::kTcTabBytes;
}
// A stage buffers: a fourth (one more half cell of lookahead between the
// dequant warps) whenever it fits next to the x tiles of this N
std::uint32_t tc_na(const spqr_layer* L, std::uint32_t N) {
    return tc_smem(L, N, 4u) + kTcStaticMax <= kSmemLimit ? 4u : 3u;
}

template <int BW, int BSZ, int HPW>
void launch_tc_hpw(const spqr_dev::TcParams& p, std::uint32_t smem, cudaStream_t st) {
    auto kern = spqr_dev::gemm_tc<BW, BSZ, BSZ, HPW>;
    static bool attr_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        cudaFuncAttributes fa{};
        ck(cudaFuncGetAttributes(&fa, kern), "cudaFuncGetAttributes(gemm_tc)");
        if (fa.sharedSizeBytes > kTcStaticMax) throw CudaError("gemm_tc: static shared memory exceeds the plan");
        ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kSmemLimit - kTcStaticMax)),
           "cudaFuncSetAttribute(gemm_tc smem)");
        attr_set[dev & 63] = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.nv);
    cfg.blockDim = dim3(spqr_dev::tc_threads(HPW));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ck(cudaLaunchKernelEx(&cfg, kern, p), "launch gemm_tc");
    ++g_launches;
}
template <int BW, int BSZ>
void launch_tc_t(const spqr_dev::TcParams& p, std::uint32_t smem, cudaStream_t st) {
    if (p.N <= static_cast<std::uint32_t>(spqr_dev::kTcHpwMaxN))
        launch_tc_hpw<BW, BSZ, 2>(p, smem, st);
    else
        launch_tc_hpw<BW, BSZ, 1>(p, smem, st);
}

void run_tc(const spqr_layer* L, const void* x, int f16, float* y, int batch, std::uint8_t* base, const WsLayout& w,
            cudaStream_t st) {
    const std::size_t esz = f16 ? 2 : 4;
    // fp32 x: hi and lo fp16 parts as two column sets of the MMA (<= 32 batch
    // columns per launch); fp16 x: <= 64
    const int per = f16 ? static_cast<int>(kTcMaxN) : static_cast<int>(kTcMaxN / 2);
    for (int b0 = 0; b0 < batch; b0 += per) {
        const std::uint32_t B = static_cast<std::uint32_t>(std::min<int>(batch - b0, per));
        const std::uint32_t Nh = f16 ? 0u : (B + 15u) & ~15u;
        const std::uint32_t N = f16 ? (B + 15u) & ~15u : 2u * Nh;
        const void* xb = static_cast<const std::uint8_t*>(x) + static_cast<std::size_t>(b0) * L->info.cols * esz;
        std::uint8_t* xpan = base + w.tc_x;
        {
            const std::uint32_t total = 2u * L->Pn * N * 16u;
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3((total + 255u) / 256u);
            cfg.blockDim = dim3(256);
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            ck(cudaLaunchKernelEx(&cfg, spqr_dev::xprep_tc, xb, f16, L->info.cols, B, N, L->Pn,
                                  static_cast<const std::uint32_t*>(L->d_order), xpan, Nh),
               "launch xprep_tc");
            ++g_launches;
        }
        spqr_dev::TcParams p{};
        p.cells = L->d_cells;
        p.cell_off = L->d_cell_off;
        p.cta_start = L->tcp.d_start;
        p.gmap = L->tcp.d_maps;
        p.cmap = L->tcp.d_maps + 2 * L->tcp.Tn;
        p.xpanels = xpan;
        p.y = y + static_cast<std::size_t>(b0) * L->info.rows;
        p.partial = reinterpret_cast<float*>(base + w.tc_part);
        p.counters = reinterpret_cast<std::uint32_t*>(base + w.tc_cnt);
        p.m = L->info.rows; p.Pn = L->Pn; p.Gn = L->Gn; p.Tn = L->tcp.Tn; p.nv = L->tcp.nv; p.B = B; p.N = N;
        p.Nh = Nh;
        p.rec_cap = L->tcp.slot_bytes; p.slot_bytes = L->tcp.slot_bytes; p.pn_magic = L->pn_magic;
        p.sigma = L->tcp.sigma;
        p.out_scale = std::ldexp(1.0f, L->tcp.sigma);
        p.na = tc_na(L, N);
        const std::uint32_t smem = tc_smem(L, N, p.na);
        switch (L->info.weight_bits * 10 + L->info.scale_bits) {
            case 22: launch_tc_t<2, 2>(p, smem, st); break;
            case 23: launch_tc_t<2, 3>(p, smem, st); break;
            case 24: launch_tc_t<2, 4>(p, smem, st); break;
            case 32: launch_tc_t<3, 2>(p, smem, st); break;
            case 33: launch_tc_t<3, 3>(p, smem, st); break;
            case 34: launch_tc_t<3, 4>(p, smem, st); break;
            case 42: launch_tc_t<4, 2>(p, smem, st); break;
            case 43: launch_tc_t<4, 3>(p, smem, st); break;
            case 44: launch_tc_t<4, 4>(p, smem, st); break;
            default: spqr::fail(spqr::Errc::config_invalid, "no gemm_tc kernel instantiated for this layer");
        }
    }
}

// ---- gemm_ex (exact mode, batch >= kExMinBatch): exact codes on the tensor cores
// below it the batch-pair gemv_cta launches are faster (tools/batch_sweep.py --exact,
// 8192x22016: batch 6 = 3 pairs, 113 us; batch 7: 141 us; one gemm_bm launch ~ 118 us)
constexpr int kExMinBatch = 7;
constexpr std::uint32_t kExMaxN = 64;  // batch columns per launch

// shared memory of one gemm_ex launch: x tile buffers + record slots
std::uint32_t ex_smem(const spqr_layer* L, std::uint32_t N, bool lo) {
    return spqr_dev::ex_nx(N) * spqr_dev::ex_xbytes(N, lo) + spqr_dev::ex_na(N) * spqr_dev::kExAOBytes +
           4u * spqr_dev::kExRecSlots * L->exp.slot_bytes;
}

void run_ex(const spqr_layer* L, const void* x, int f16, float* y, int batch, std::uint8_t* base, const WsLayout& w,
            cudaStream_t st) {
    const std::size_t esz = f16 ? 2 : 4;
    const bool lo = !f16;
    // batch columns per launch: 64, or 32 when the fp32-x tiles of N = 64 do not fit next to the records
    const int per = ex_smem(L, 64, lo) + spqr_dev::kExStaticMax <= kSmemLimit ? 64 : 32;
    for (int b0 = 0; b0 < batch; b0 += per) {
        const std::uint32_t B = static_cast<std::uint32_t>(std::min<int>(batch - b0, per));
        const std::uint32_t N = B <= 16 ? 16u : (B <= 32 ? 32u : 64u);
        const std::uint32_t xb = spqr_dev::ex_xbytes(N, lo);
        const void* xs = static_cast<const std::uint8_t*>(x) + static_cast<std::size_t>(b0) * L->info.cols * esz;
        std::uint8_t* xpan = base + w.ex_x;
        float* esc = reinterpret_cast<float*>(base + w.ex_scale);
        {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(N, std::max(1u, 256u / N));
            cfg.blockDim = dim3(256);
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            ck(cudaLaunchKernelEx(&cfg, spqr_dev::xprep_ex, xs, f16, L->info.cols, B, N, L->Pn,
                                  static_cast<const std::uint32_t*>(L->d_order), xpan, esc, xb, lo ? 1u : 0u,
                                  static_cast<int>(L->info.weight_bits)),
               "launch xprep_ex");
            ++g_launches;
        }
        spqr_dev::ExParams p{};
        p.cells = L->d_cells;
        p.cell_off = L->d_cell_off;
        p.cta_start = L->tcp.d_start;
        p.gmap = L->tcp.d_maps;
        p.cmap = L->tcp.d_maps + 2 * L->tcp.Tn;
        p.xpanels = xpan;
        p.escale = esc;
        p.y = y + static_cast<std::size_t>(b0) * L->info.rows;
        p.partial = reinterpret_cast<float*>(base + w.tc_part);
        p.counters = reinterpret_cast<std::uint32_t*>(base + w.tc_cnt);
        p.m = L->info.rows; p.Pn = L->Pn; p.Gn = L->Gn; p.Tn = L->tcp.Tn; p.nv = L->tcp.nv; p.B = B; p.N = N;
        p.rec_cap = L->exp.slot_bytes; p.slot_bytes = L->exp.slot_bytes; p.pn_magic = L->pn_magic;
        p.lo = lo ? 1u : 0u;
        p.xb = xb;
        ck(spqr_dev::launch_gemm_ex(static_cast<int>(L->info.weight_bits), static_cast<int>(L->info.scale_bits),
                                    static_cast<int>(N), p, ex_smem(L, N, lo), kSmemLimit, st),
           "launch gemm_ex");
        ++g_launches;
    }
}

// ---- gemm_bm (exact mode): batch in the mma.sync M dimension, chunks of <= 32 columns
std::uint32_t bm_smem(const spqr_layer* L, std::uint32_t N) {
    return spqr_dev::bm_nx(N) * spqr_dev::bm_xbytes(N) + spqr_dev::bm_fixed_smem(N) +
           4u * spqr_dev::kBmRecSlots * L->exp.slot_bytes;
}

void run_bm(const spqr_layer* L, const void* x, int f16, float* y, int batch, std::uint8_t* base, const WsLayout& w,
            cudaStream_t st) {
    if (!f16) spqr::fail(spqr::Errc::config_invalid, "gemm_bm: fp16 x only");
    for (int b0 = 0; b0 < batch; b0 += 32) {
        const std::uint32_t B = static_cast<std::uint32_t>(std::min(batch - b0, 32));
        const int mt = B <= 16 ? 1 : 2;
        const std::uint32_t N = 16u * static_cast<std::uint32_t>(mt);
        const void* xs = static_cast<const std::uint8_t*>(x) + static_cast<std::size_t>(b0) * L->info.cols * 2;
        std::uint8_t* xpan = base + w.ex_x;
        float* esc = reinterpret_cast<float*>(base + w.ex_scale);
        {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(N, std::max(1u, 256u / N));
            cfg.blockDim = dim3(256);
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            ck(cudaLaunchKernelEx(&cfg, spqr_dev::xprep_bm, xs, 1, L->info.cols, B, N, L->Pn,
                                  static_cast<const std::uint32_t*>(L->d_order), xpan, esc,
                                  static_cast<int>(L->info.weight_bits)),
               "launch xprep_bm");
            ++g_launches;
        }
        spqr_dev::ExParams p{};
        p.cells = L->d_cells;
        p.cell_off = L->d_cell_off;
        p.cta_start = L->tcp.d_start;
        p.gmap = L->tcp.d_maps;
        p.cmap = L->tcp.d_maps + 2 * L->tcp.Tn;
        p.xpanels = xpan;
        p.escale = esc;
        p.y = y + static_cast<std::size_t>(b0) * L->info.rows;
        p.partial = reinterpret_cast<float*>(base + w.tc_part);
        p.counters = reinterpret_cast<std::uint32_t*>(base + w.tc_cnt);
        p.m = L->info.rows; p.Pn = L->Pn; p.Gn = L->Gn; p.Tn = L->tcp.Tn; p.nv = L->tcp.nv; p.B = B; p.N = N;
        p.rec_cap = L->exp.slot_bytes; p.slot_bytes = L->exp.slot_bytes; p.pn_magic = L->pn_magic;
        p.usplit = L->d_usplit;
        ck(spqr_dev::launch_gemm_bm(static_cast<int>(L->info.weight_bits), static_cast<int>(L->info.scale_bits), mt, p,
                                    bm_smem(L, N), kSmemLimit, st),
           "launch gemm_bm");
        ++g_launches;
    }
}

// gemv_cta launch parameters for one batch column
spqr_dev::CtaParams cta_params(const spqr_layer* L, const void* x, int xm, float* y, std::uint8_t* base,
                               const WsLayout& w) {
    const auto& c = L->cta[xm];
    spqr_dev::CtaParams p{};
    p.cells = L->d_cells;
    p.cell_off = L->d_cell_off;
    p.cta_start = c.d_start;
    p.x = x;
    p.order = static_cast<const std::uint32_t*>(L->d_order);
    p.y = y;
    p.xpart = reinterpret_cast<float*>(base + w.xpart);
    p.xcnt = reinterpret_cast<std::uint32_t*>(base + w.xcnt);
    p.m = L->info.rows; p.n = L->info.cols; p.Pn = L->Pn; p.Gn = L->Gn; p.nvcta = c.nvcta;
    p.pn_magic = L->pn_magic;
    p.rec_cap = c.rec_cap; p.slot_bytes = c.slot_bytes;
    p.pan_off = c.pan_off; p.part_off = c.part_off; p.off_off = c.off_off; p.gd_off = c.gd_off;
    p.part_cap = c.part_cap;
    p.first_rec = reinterpret_cast<const uint2*>(c.d_first);
    if (c.grid < static_cast<std::uint32_t>(spqr_dev::kQFirst))
        std::copy(c.h_start.begin(), c.h_start.begin() + c.grid + 1, p.q_first);
    // 16-B vector loads of x: unpermuted, aligned (batch pair: the second
    // column, n halves further on, too)
    p.x_vec = (!p.order && (reinterpret_cast<std::uintptr_t>(p.x) & 15u) == 0 &&
               (xm != 2 || (2ull * L->info.cols) % 16u == 0))
                  ? 1u
                  : 0u;
    return p;
}

// stage: 0 = x preparation + product, 1 = x preparation only, 2 = product only
// (reuses the workspace the last stage-1 call prepared; used to time the hot
// kernel alone).
void run_matvec(const spqr_layer* L, const void* x, int dtype, float* y, int batch, void* ws, std::uint64_t wsb,
                cudaStream_t st, int stage = 0) {
    if (batch < 1) spqr::fail(spqr::Errc::shape_mismatch, "batch must be >= 1");
    if (dtype != SPQR_F16 && dtype != SPQR_F32) spqr::fail(spqr::Errc::config_invalid, "x dtype must be f16 or f32");
    const WsLayout w = ws_layout(L, batch);
    if (wsb < w.total) spqr::fail(spqr::Errc::config_invalid, "workspace too small");
    auto* base = static_cast<std::uint8_t*>(ws);
    const int f16 = dtype == SPQR_F16;
    if (L->fast && L->exact && L->exp.ok && batch >= kExMinBatch) {
        if (stage == 1) return;
        // fp16 x up to 32 columns: batch in the mma.sync M dimension (gemm_bm); fp32 x and wider
        // batches: per-block accumulators on tcgen05 (gemm_ex; 64 columns per launch)
        if (f16 && batch <= 32) run_bm(L, x, f16, y, batch, base, w, st);
        else run_ex(L, x, f16, y, batch, base, w, st);
        return;
    }
    if (L->fast && !L->exact && batch >= kTcMinBatch) {
        if (stage == 1) return;
        run_tc(L, x, f16, y, batch, base, w, st);
        return;
    }
    if (L->fast) {
        // one fused launch per batch column (x preparation happens inside)
        if (stage == 1) return;
        // fp16 x: batch columns two at a time through the batch-pair kernel
        // (each weight decoded once for both), an odd last column alone
        const std::size_t esz = f16 ? 2 : 4;
        for (int b = 0; b < batch;) {
            const int xm = !f16 ? 1 : (b + 1 < batch ? 2 : 0);
            spqr_dev::CtaParams p = cta_params(L, static_cast<const std::uint8_t*>(x) +
                                                      static_cast<std::size_t>(b) * L->info.cols * esz,
                                               xm, y + static_cast<std::size_t>(b) * L->info.rows, base, w);
            dispatch_cta(p, L, xm, st);
            b += xm == 2 ? 2 : 1;
        }
    } else {
        auto* xp = reinterpret_cast<float*>(base + w.xp);
        const std::uint64_t nx = static_cast<std::uint64_t>(L->info.cols) * batch;
        if (stage != 2) {
            spqr_dev::xprep_raw<<<static_cast<unsigned>((nx + 255) / 256), 256, 0, st>>>(x, f16, L->info.cols,
                                                                                      batch, L->d_order, xp);
            ck(cudaGetLastError(), "launch xprep_raw");
            ++g_launches;
        }
        if (stage == 1) return;
        const spqr_dev::RawGeom geo = raw_geom(L);
        for (int b = 0; b < batch; ++b) {
            spqr_dev::gemv_raw<<<(L->info.rows + 7) / 8, 256, 0, st>>>(
                geo, xp + static_cast<std::size_t>(b) * L->info.cols, y + static_cast<std::size_t>(b) * L->info.rows);
            ck(cudaGetLastError(), "launch gemv_raw");
            ++g_launches;
        }
    }
}

// A handle-owned workspace, zero-filled (the kernels return the exchange
// words and counters to zero).  Growing it syncs the device first: an
// in-flight launch may still use the old one.
void ensure_ws(const spqr_layer* L, int batch, void*& ws, std::uint64_t& bytes) {
    const std::uint64_t need = ws_layout(L, batch).total;
    if (bytes >= need) return;
    if (ws) {
        ck(cudaDeviceSynchronize(), "sync before workspace growth");
        cudaFree(ws);
        ws = nullptr;
        bytes = 0;
    }
    ws = dalloc<std::uint8_t>(need);
    ck(cudaMemset(ws, 0, need), "zero workspace");
    bytes = need;
}
void ensure_own_ws(const spqr_layer* L, int batch) { ensure_ws(L, batch, L->d_ws, L->ws_bytes); }

// gemv_cta partition: contiguous cell ranges balanced by bytes (record bytes +
// a per-cell fixed cost), one range per CTA -- or several per CTA when the
// per-range row-sum array would not fit shared memory.  Every range holds at
// least Pn cells (a row-group pair is shared by at most two ranges; the
// kernel's pair exchange relies on it); layers with fewer pairs than SMs get
// one whole pair per range.  Plus the shared-memory plan: two record slots
// per warp, per-warp x panels, the row-sum array, record offsets, pair counts.
void plan_cta(spqr_layer* L, const spqr::detail::TiledHost& t, int sms, int xi) {
    auto& c = L->cta[xi];
    const std::uint32_t Q = t.Gn * t.Pn;
    const std::uint32_t cellb = t.cell_bytes;
    const std::uint32_t panel = spqr_tiled::panel_bytes(xi);
    const std::uint32_t ncol = xi == 2 ? 2u : 1u;  // row sums per cell: 32 per batch column
    const std::uint32_t budget = kSmemLimit - kCtaStaticMax;
    constexpr std::uint32_t kPartMax = 48u * 1024u;  // row-sum array cap
    const std::uint32_t S = static_cast<std::uint32_t>(sms);
    std::vector<double> pre(Q + 1, 0.0);
    for (std::uint32_t q = 0; q < Q; ++q) pre[q + 1] = pre[q] + 512.0 + (t.cell_off[q + 1] - t.cell_off[q]);
    std::vector<std::uint32_t> st;
    std::uint32_t mc = 0;
    auto cut = [&](std::uint32_t nv) {  // byte-balanced cut; false if a range is shorter than Pn
        st.assign(nv + 1, Q);
        std::uint32_t q = 0;
        for (std::uint32_t k = 0; k < nv; ++k) {
            const double target = pre[Q] * k / nv;
            while (q < Q && pre[q] + 0.5 * (pre[q + 1] - pre[q]) < target) ++q;
            st[k] = q;
        }
        st[nv] = Q;
        mc = 0;
        bool ok = true;
        for (std::uint32_t k = 0; k < nv; ++k) {
            mc = std::max(mc, st[k + 1] - st[k]);
            ok = ok && st[k + 1] - st[k] >= t.Pn;
        }
        return ok;
    };
    // x panels once per CTA (all Pn in shared memory) whenever the two record
    // slots per warp still hold a cell plus ~256 outliers next to them; else
    // each warp builds its cell's panel.  fp32 x / batch-pair panels are 2128 /
    // 1712 B: for them the slots need only hold 90 % of the layer's records
    // whole (a per-warp panel build costs ~15 % per cell, a record's outliers
    // beyond its slot are a few global loads)
    std::uint32_t rec90 = cellb;
    if (Q) {
        std::vector<std::uint32_t> rs(Q);
        for (std::uint32_t q = 0; q < Q; ++q) rs[q] = t.cell_off[q + 1] - t.cell_off[q];
        const std::size_t k = static_cast<std::size_t>(0.9 * (Q - 1));
        std::nth_element(rs.begin(), rs.begin() + k, rs.end());
        rec90 = rs[k];
    }
    const std::uint32_t shx_bytes = t.Pn * panel;
    auto fixed_of = [&](std::uint32_t cap) {  // row-sum array + record offsets + pair counts
        return ((cap * 128u * ncol + 127u) & ~127u) + (((cap + 9u) * 4u + 127u) & ~127u) +
               (((cap + 1u) * 4u + 127u) & ~127u);
    };
    auto shx_fits = [&](std::uint32_t cap) {
        const std::uint32_t fixed = fixed_of(std::max<std::uint32_t>(cap, 1));
        if (t.Pn > 64u || shx_bytes + fixed >= budget) return false;  // 64: the kernel's panel-ready flags
        const std::uint32_t shx_slot = ((budget - shx_bytes - fixed) / (2u * kNC)) & ~127u;
        return shx_slot >= cellb + 16u && (shx_bytes <= 40u * 1024u || shx_slot >= cellb + 1024u ||
                                           shx_slot >= std::max(cellb + 256u, rec90));
    };
    std::uint32_t nv = 0;
    if (t.Gn <= S) {  // one whole pair per range
        nv = t.Gn;
        st.resize(nv + 1);
        for (std::uint32_t k = 0; k <= nv; ++k) st[k] = k * t.Pn;
        mc = t.Pn;
    } else {
        nv = S;
        while (!cut(nv) && nv > 1) --nv;
        while (mc * 128u * ncol > kPartMax) {  // more ranges than SMs: several per CTA
            std::uint32_t nn = nv + S;
            while (!cut(nn) && nn > nv + 1) --nn;
            nv = nn;
        }
        // fp32-x panels: a second range per CTA when its halved row-sum array
        // is what lets the panels into shared memory (44032x8192 fp32: 298 ->
        // 149 cells per range, 55.3 -> 53.5 us; batch-pair layers measured
        // slower that way: 37.1 -> 38.5 us on 22016x8192)
        if (xi == 1 && !shx_fits(mc)) {
            const std::uint32_t nv0 = nv;
            std::uint32_t nn = nv + S;
            bool ok = false;
            while (!(ok = cut(nn)) && nn > nv + 1) --nn;
            if (ok && shx_fits(mc))
                nv = nn;
            else
                cut(nv0);
        }
    }
    c.nvcta = nv;
    c.grid = std::min<std::uint32_t>(nv, S);
    c.part_cap = std::max<std::uint32_t>(mc, 1);
    const std::uint32_t part_bytes = (c.part_cap * 128u * ncol + 127u) & ~127u;
    const std::uint32_t off_bytes = ((c.part_cap + 9u) * 4u + 127u) & ~127u;  // 16-B aligned superset
    const std::uint32_t gd_bytes = ((c.part_cap + 1u) * 4u + 127u) & ~127u;
    c.shared_x = shx_fits(c.part_cap);
    const std::uint32_t pan_bytes = c.shared_x ? shx_bytes : kNC * panel;
    const std::uint32_t ring_avail = budget - pan_bytes - part_bytes - off_bytes - gd_bytes;
    // two record slots per warp; outliers beyond a slot are read from HBM
    const std::uint32_t slot = std::min((ring_avail / (2u * kNC)) & ~127u, (cellb + 4096u + 127u) & ~127u);
    if (slot < cellb + 16u)
        spqr::fail(spqr::Errc::config_invalid,
                   "gemv_cta: shared memory plan does not fit (x mode " + std::to_string(xi) + ", record slot " +
                       std::to_string(slot) + " B < cell " + std::to_string(cellb) + " B + 16)");
    c.slot_bytes = slot;
    c.rec_cap = slot;
    c.pan_off = slot * 2u * kNC;
    c.part_off = c.pan_off + pan_bytes;
    c.off_off = c.part_off + part_bytes;
    c.gd_off = c.off_off + off_bytes;
    c.smem = c.gd_off + gd_bytes;
    c.d_start = dalloc<std::uint32_t>(st.size());
    ck(cudaMemcpy(c.d_start, st.data(), 4 * st.size(), cudaMemcpyHostToDevice), "H2D cta_start");
    c.h_start = st;
    // CTA v's first range is range v; its warp w takes cell w first
    std::vector<std::uint32_t> first(2ull * c.grid * kNC, 0u);
    for (std::uint32_t v = 0; v < c.grid; ++v)
        for (std::uint32_t w = 0; w < static_cast<std::uint32_t>(kNC); ++w) {
            const std::uint32_t q = st[v] + w;
            if (q < st[v + 1]) {
                first[2 * (v * kNC + w)] = t.cell_off[q];
                first[2 * (v * kNC + w) + 1] = t.cell_off[q + 1];
            }
        }
    c.d_first = dalloc<std::uint32_t>(first.size());
    ck(cudaMemcpy(c.d_first, first.data(), 4 * first.size(), cudaMemcpyHostToDevice), "H2D first records");
    if (xi == 0) {  // q / Pn as a multiply-high (Pn == 1: the kernel uses q itself)
        const std::uint64_t mg = t.Pn > 1 ? ((1ull << 32) + t.Pn - 1) / t.Pn : 0;
        L->pn_magic = static_cast<std::uint32_t>(mg);
        if (t.Pn > 1)
            for (std::uint64_t q = 0; q <= Q; ++q)
                if (((q * mg) >> 32) != q / t.Pn)
                    spqr::fail(spqr::Errc::config_invalid, "gemv_cta: cell index division out of range");
    }
}

// gemm_tc partition: units (128-row tile T, panel P), T-major, cut into
// byte-balanced contiguous ranges (one per CTA); tiles shared by several
// ranges are reduced through partial slots in range order.  sigma: the
// per-layer power of two that keeps s * 2^(24 - p - sigma) < 2^15 for every
// first-level scale s (binary16 range of the dequantization multiplier).
void plan_tc(spqr_layer* L, const spqr::detail::TiledHost& t, const std::vector<spqr::detail::StreamView>& views,
             int sms) {
    auto& c = L->tcp;
    c.Tn = (t.Gn + 3u) / 4u;
    const std::uint32_t U = c.Tn * t.Pn;
    std::vector<double> pre(U + 1, 0.0);
    for (std::uint32_t u = 0; u < U; ++u) {
        const std::uint32_t T_ = u / t.Pn, P = u % t.Pn;
        double b = 2048.0;
        for (std::uint32_t i = 0; i < 4; ++i) {
            const std::uint32_t G = 4 * T_ + i;
            if (G < t.Gn) b += t.cell_off[G * t.Pn + P + 1] - t.cell_off[G * t.Pn + P];
        }
        pre[u + 1] = pre[u] + b;
    }
    const std::uint32_t nv = std::max<std::uint32_t>(1, std::min<std::uint32_t>(static_cast<std::uint32_t>(sms), U));
    std::vector<std::uint32_t> st(nv + 1, U);
    std::uint32_t q = 0;
    for (std::uint32_t k = 0; k < nv; ++k) {
        const double target = pre[U] * k / nv;
        while (q < U && pre[q] + 0.5 * (pre[q + 1] - pre[q]) < target) ++q;
        st[k] = q;
    }
    st[nv] = U;
    c.nv = nv;
    std::vector<std::uint32_t> gmap(2ull * c.Tn, 0), cmap(2ull * nv, 0);
    for (std::uint32_t k = 0; k < nv; ++k) {
        const std::uint32_t a = st[k], b = st[k + 1];
        if (a >= b) continue;
        const std::uint32_t ta = a / t.Pn, tb = (b - 1) / t.Pn;
        const bool whole_a = a == ta * t.Pn && (tb != ta || b == (ta + 1) * t.Pn);
        if (!whole_a) cmap[2 * k] = gmap[2 * ta + 1]++;
        if (tb != ta && b != (tb + 1) * t.Pn) cmap[2 * k + 1] = gmap[2 * tb + 1]++;
    }
    std::uint32_t slots = 0;
    for (std::uint32_t T_ = 0; T_ < c.Tn; ++T_) {
        gmap[2 * T_] = slots;
        slots += gmap[2 * T_ + 1];
    }
    c.pslots = slots;
    c.slot_bytes = (t.cell_bytes + 512u + 127u) & ~127u;  // outliers beyond a slot are read from HBM
    const std::uint32_t need = 3u * 128u * 128u * 2u + 3u * 256u * kTcMaxN + 8u * c.slot_bytes + spqr_dev::kTcTabBytes;
    if (need + kTcStaticMax > kSmemLimit)
        c.slot_bytes = ((kSmemLimit - kTcStaticMax - (need - 8u * c.slot_bytes)) / 8u) & ~127u;
    if (c.slot_bytes < t.cell_bytes + 16u) spqr::fail(spqr::Errc::config_invalid, "gemm_tc: shared memory plan");
    // sigma from the first-level scale bound
    double smax = 0.0;
    for (const auto& v : views) {
        const int top = (1 << v.sb) - 1;
        for (std::uint32_t k = 0; k < v.nblocks; ++k)
            for (std::uint32_t g = 0; g < v.ngroups; ++g) {
                const std::size_t o = v.record_offset(k, g);
                const double S = spqr::fp16_to_float(spqr::detail::StreamView::load_u16(v.base + o));
                const double Z = spqr::fp16_to_float(spqr::detail::StreamView::load_u16(v.base + o + 2));
                smax = std::max({smax, std::fabs(S * (0 - Z)), std::fabs(S * (top - Z))});
            }
    }
    c.sigma = 0;
    // weights w 2^-sigma up to ~2^12 (s (q - z) <= ~8 smax): binary16 normals
    // for the whole useful range, no subnormal underflow of small weights
    if (smax > 0 && std::isfinite(smax)) c.sigma = std::clamp(static_cast<int>(std::ceil(std::log2(smax))) - 9, -100, 100);
    c.d_start = dalloc<std::uint32_t>(st.size());
    c.d_maps = dalloc<std::uint32_t>(gmap.size() + cmap.size());
    ck(cudaMemcpy(c.d_start, st.data(), 4 * st.size(), cudaMemcpyHostToDevice), "H2D tc start");
    ck(cudaMemcpy(c.d_maps, gmap.data(), 4 * gmap.size(), cudaMemcpyHostToDevice), "H2D tc gmap");
    ck(cudaMemcpy(c.d_maps + gmap.size(), cmap.data(), 4 * cmap.size(), cudaMemcpyHostToDevice), "H2D tc cmap");
}

// gemm_ex: the outlier bound and the shared-memory plan (ranges: plan_tc's).
void plan_ex(spqr_layer* L, const spqr::detail::TiledHost& t, const std::vector<spqr::detail::StreamView>& views) {
    auto& e = L->exp;
    e.ok = false;
    float vmax = 0.0f;
    for (const auto& v : views) {
        if (v.ent_off + 4ull * v.nnz > v.nbytes) return;
        for (std::uint32_t i = 0; i < v.nnz; ++i) vmax = std::max(vmax, std::fabs(spqr::fp16_to_float(v.ent_val(i))));
    }
    // fp16(v 2^p_c) exact for p_c <= 7 when |v| 2^7 <= 65504
    if (!(vmax < 512.0f)) return;
    e.slot_bytes = (t.cell_bytes + 512u + 127u) & ~127u;  // outliers beyond a slot are read from HBM
    // the largest plan that must fit: N = 32 with fp32 x (N = 64 falls back to two 32-column launches)
    const std::uint32_t base = spqr_dev::ex_nx(32) * spqr_dev::ex_xbytes(32, true) +
                               spqr_dev::ex_na(32) * spqr_dev::kExAOBytes + spqr_dev::kExStaticMax;
    const std::uint32_t nslot = 4u * spqr_dev::kExRecSlots;
    if (base + nslot * e.slot_bytes > kSmemLimit) e.slot_bytes = ((kSmemLimit - base) / nslot) & ~127u;
    if (e.slot_bytes < t.cell_bytes + 16u) return;
    const std::uint32_t ncell = t.Gn * t.Pn;
    L->d_usplit = dalloc<std::uint32_t>(ncell);
    spqr_dev::cell_unit_split<<<(ncell + 255) / 256, 256>>>(L->d_cells, L->d_cell_off, ncell, t.cell_bytes, L->d_usplit);
    ck(cudaGetLastError(), "launch cell_unit_split");
    ck(cudaDeviceSynchronize(), "cell_unit_split");
    e.ok = true;
}

// Every launch plan of a tiled layer (geometry + record offsets in t).
void make_plans(spqr_layer* L, const spqr::detail::TiledHost& t, const std::vector<spqr::detail::StreamView>& views) {
    L->Gn = t.Gn; L->Pn = t.Pn; L->cell_bytes = t.cell_bytes; L->n_pad = t.Pn * 256;
    int sms = 0;
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, L->device), "SM count");
    plan_cta(L, t, sms, 0);
    plan_cta(L, t, sms, 1);
    plan_cta(L, t, sms, 2);
    plan_tc(L, t, views, sms);
    plan_ex(L, t, views);
}

// Host-built tiled layer (transcode.cpp) -> HBM + plans; returns device bytes.
std::uint64_t upload_tiled(spqr_layer* L, const spqr::detail::TiledHost& t,
                           const std::vector<spqr::detail::StreamView>& views) {
    L->d_cells = dalloc<std::uint8_t>(t.cells.size() + 16);
    ck(cudaMemcpy(L->d_cells, t.cells.data(), t.cells.size(), cudaMemcpyHostToDevice), "H2D cells");
    L->d_cell_off = dalloc<std::uint32_t>(t.cell_off.size() + 4);  // + 4: gemv_cta copies 16-B aligned supersets
    ck(cudaMemcpy(L->d_cell_off, t.cell_off.data(), 4 * t.cell_off.size(), cudaMemcpyHostToDevice), "H2D cell_off");
    make_plans(L, t, views);
    return t.cells.size() + 4 * t.cell_off.size();
}

// Device-built tiled layer (transcode_dev.cuh, byte-identical to the host
// transcode) from streams already resident on the device: per-cell outlier
// counts on the GPU, record offsets prefixed on the host, then the unit and
// entry kernels write the cells in place.  Several streams stack row-wise.
std::uint64_t transcode_on_device(spqr_layer* L, const std::vector<spqr::detail::StreamView>& views,
                                  const std::vector<const std::uint8_t*>& d_streams) {
    spqr::detail::TiledHost t;
    const auto& v0 = views[0];
    t.Pn = (v0.cols + 255) / 256;
    t.cell_bytes = spqr_tiled::cell_bytes(v0.wb, v0.sb, v0.zb);
    t.prefix.assign(v0.base, v0.base + v0.rec_off);
    std::vector<std::uint32_t> gbase;  // first cell row of each member
    std::vector<spqr_dev::RawGeom> geos;
    for (std::size_t i = 0; i < views.size(); ++i) {
        gbase.push_back(t.Gn);
        t.Gn += (views[i].rows + 31) / 32;
        geos.push_back(raw_geom_of(views[i], d_streams[i], nullptr));
    }
    const std::size_t ncell = static_cast<std::size_t>(t.Gn) * t.Pn;
    std::uint32_t* d_cnt = dalloc<std::uint32_t>(ncell);
    for (std::size_t i = 0; i < views.size(); ++i) {
        const std::uint32_t gn = (views[i].rows + 31) / 32, cells_i = gn * t.Pn;
        spqr_dev::tc_entries<true><<<(cells_i * 32 + 255) / 256, 256>>>(
            geos[i], gn, t.Pn, t.cell_bytes, nullptr, nullptr, d_cnt + static_cast<std::size_t>(gbase[i]) * t.Pn);
        ck(cudaGetLastError(), "launch tc_entries<count>");
    }
    std::vector<std::uint32_t> cnt(ncell);
    ck(cudaMemcpy(cnt.data(), d_cnt, 4 * ncell, cudaMemcpyDeviceToHost), "D2H outlier counts");
    cudaFree(d_cnt);
    t.cell_off.assign(ncell + 1, 0);
    std::uint64_t total = 0;
    for (std::size_t q = 0; q < ncell; ++q) {
        t.cell_off[q] = static_cast<std::uint32_t>(total);
        total += t.cell_bytes + 16ull * ((cnt[q] + 3) / 4);
        if (total > 0xfffffff0ull) spqr::fail(spqr::Errc::config_invalid, "layer too large for 32-bit record offsets");
    }
    t.cell_off[ncell] = static_cast<std::uint32_t>(total);
    L->d_cells = dalloc<std::uint8_t>(total + 16);
    L->d_cell_off = dalloc<std::uint32_t>(t.cell_off.size() + 4);  // + 4: gemv_cta copies 16-B aligned supersets
    ck(cudaMemcpy(L->d_cell_off, t.cell_off.data(), 4 * t.cell_off.size(), cudaMemcpyHostToDevice), "H2D cell_off");
    for (std::size_t i = 0; i < views.size(); ++i) {
        const std::uint32_t gn = (views[i].rows + 31) / 32;
        const std::uint32_t* off_i = L->d_cell_off + static_cast<std::size_t>(gbase[i]) * t.Pn;
        const unsigned ub = (2u * gn * t.Pn * 32u + 255u) / 256u;
        switch (v0.wb) {
            case 2: spqr_dev::tc_units<2><<<ub, 256>>>(geos[i], gn, t.Pn, off_i, L->d_cells); break;
            case 3: spqr_dev::tc_units<3><<<ub, 256>>>(geos[i], gn, t.Pn, off_i, L->d_cells); break;
            default: spqr_dev::tc_units<4><<<ub, 256>>>(geos[i], gn, t.Pn, off_i, L->d_cells); break;
        }
        ck(cudaGetLastError(), "launch tc_units");
        spqr_dev::tc_entries<false><<<(gn * t.Pn * 32 + 255) / 256, 256>>>(geos[i], gn, t.Pn, t.cell_bytes, off_i,
                                                                          L->d_cells, nullptr);
        ck(cudaGetLastError(), "launch tc_entries");
    }
    ck(cudaDeviceSynchronize(), "device transcode");
    make_plans(L, t, views);
    return total + 4 * t.cell_off.size();
}
}  // namespace

// Fused all-gather target of one rank: one cudaMalloc'd block (exported to
// the other ranks by CUDA IPC): [0, 32) per-source-rank round counters,
// [64] this rank's round, [68] CTAs done (local), [128, 160) per-source-rank
// latest started round (a peer's band kernel posts it before anyone stores
// that round into its y), [256, ...) the full y.
struct spqr_gather {
    int device = 0, world = 1, rank = 0;
    std::uint32_t rows = 0;
    std::uint8_t* base = nullptr;
    std::uint8_t* peer[spqr_dev::kMaxPeers + 1] = {};  // by rank (own block at [rank])
    std::uint32_t row_base[spqr_dev::kMaxPeers + 1] = {};
    bool open = false;
    static constexpr std::size_t kY = 256;
    float* y() const { return reinterpret_cast<float*>(base + kY); }
    ~spqr_gather() {
        for (int j = 0; j < world; ++j)
            if (j != rank && peer[j]) cudaIpcCloseMemHandle(peer[j]);
        if (base) cudaFree(base);
    }
};

// ================================================================ C ABI ====
extern "C" {

int spqr_layer_create(const uint8_t* stream, size_t nbytes, const spqr_layer_opts* opts, spqr_layer** out) {
    *out = nullptr;
    return guard([&] {
        spqr_layer_opts o{};
        o.device = -1;
        if (opts) o = *opts;
        std::vector<std::uint8_t> band;
        const std::uint8_t* s = stream;
        std::size_t n = nbytes;
        if ((o.row_begin != 0 || o.row_end != 0) && o.row_end <= o.row_begin)
            spqr::fail(spqr::Errc::config_invalid, "row band must be non-empty (0, 0 = all rows)");
        if (o.row_end > o.row_begin) {
            band = spqr::slice_rows(std::span<const std::uint8_t>(stream, nbytes), o.row_begin, o.row_end);
            s = band.data();
            n = band.size();
        }
        const spqr::detail::StreamView v = spqr::detail::parse_stream(s, n);
        int ndev = 0;
        ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
        if (ndev == 0) throw CudaError("CUDA: no device");
        DevGuard dg(o.device);
        auto L = std::make_unique<spqr_layer>();
        ck(cudaGetDevice(&L->device), "cudaGetDevice");
        L->prefix.assign(s, s + v.rec_off);
        L->geo = spqr::detail::geometry_from_prefix(L->prefix.data(), L->prefix.size());
        std::memset(&L->info, 0, sizeof(L->info));
        L->info.rows = v.rows; L->info.cols = v.cols; L->info.weight_bits = v.wb;
        L->info.scale_bits = v.sb; L->info.zero_bits = v.zb; L->info.beta1 = v.b1; L->info.beta2 = v.b2;
        L->info.outlier_count = v.nnz; L->info.flags = v.flags; L->info.has_permutation = v.has_permutation;
        L->info.tau = v.tau; L->info.lambda_rel = v.lambda_rel;
        L->info.payload_bytes = n - spqr::kSpqrHeaderBytes;
        L->info.device = L->device;
        std::uint64_t dev_bytes = 0;

        if (v.has_permutation) {
            std::vector<std::uint32_t> ord(v.cols);
            for (std::uint32_t k = 0; k < v.cols; ++k) ord[k] = v.order(k);
            L->d_order = dalloc<std::uint32_t>(v.cols);
            ck(cudaMemcpy(L->d_order, ord.data(), 4ull * v.cols, cudaMemcpyHostToDevice), "H2D order");
            dev_bytes += 4ull * v.cols;
        }
        L->fast = !o.force_generic && spqr::detail::tiled_supported(v);
        // the raw stream stays in HBM only for the generic kernels (or on
        // request); a fast-path layer's stream visits the device for the
        // transcode and is freed -- matvec, dequantize and export read cells
        const bool keep = !L->fast || o.keep_stream;
        if (keep || (L->fast && !o.host_transcode)) {
            L->d_stream = dalloc<std::uint8_t>(n + 16);
            ck(cudaMemcpy(L->d_stream, s, n, cudaMemcpyHostToDevice), "H2D stream");
        }
        if (L->fast)
            dev_bytes += o.host_transcode ? upload_tiled(L.get(), spqr::detail::transcode_to_tiled(v, 0), {v})
                                          : transcode_on_device(L.get(), {v}, {L->d_stream});
        if (keep) {
            dev_bytes += n;
        } else if (L->d_stream) {
            cudaFree(L->d_stream);
            L->d_stream = nullptr;
        }
        L->info.fast_path = L->fast;
        ensure_own_ws(L.get(), 1);
        dev_bytes += L->ws_bytes;
        L->info.device_bytes = dev_bytes;
        *out = L.release();
    });
}

// Extension (no reference counterpart: the reference decodes one tensor at a
// time): several layers with the same input -- q/k/v, or gate/up -- stacked
// row-wise into one handle, so one launch computes all their outputs (rows of
// layer i follow those of layer i-1 in y).  Every stream must be on the fast
// path with identical columns, widths, group sizes and permutation, and all
// but the last must have rows % 32 == 0.  matvec only: dequantize / export
// on a stacked handle return SPQR_E_CONFIG_INVALID.
int spqr_layer_create_stacked(const uint8_t* const* streams, const size_t* sizes, int count,
                              const spqr_layer_opts* opts, spqr_layer** out) {
    *out = nullptr;
    return guard([&] {
        if (count < 1 || !streams || !sizes) spqr::fail(spqr::Errc::config_invalid, "stacked: no layers");
        spqr_layer_opts o{};
        o.device = -1;
        if (opts) o = *opts;
        if (o.row_end > o.row_begin || o.force_generic)
            spqr::fail(spqr::Errc::config_invalid, "stacked: row bands / generic path not supported");
        std::vector<spqr::detail::StreamView> views;
        for (int i = 0; i < count; ++i) views.push_back(spqr::detail::parse_stream(streams[i], sizes[i]));
        const auto& v0 = views[0];
        for (int i = 0; i < count; ++i) {
            const auto& v = views[i];
            if (!spqr::detail::tiled_supported(v))
                spqr::fail(spqr::Errc::config_invalid, "stacked: layer outside the tiled geometry");
            if (v.cols != v0.cols || v.wb != v0.wb || v.sb != v0.sb || v.zb != v0.zb || v.b1 != v0.b1 ||
                v.b2 != v0.b2 || v.has_permutation != v0.has_permutation)
                spqr::fail(spqr::Errc::shape_mismatch, "stacked: layers differ in columns, widths or groups");
            if (i + 1 < count && v.rows % 32 != 0)
                spqr::fail(spqr::Errc::shape_mismatch, "stacked: rows of all but the last layer must be a multiple of 32");
            if (v.has_permutation)
                for (std::uint32_t k = 0; k < v.cols; ++k)
                    if (v.order(k) != v0.order(k)) spqr::fail(spqr::Errc::shape_mismatch, "stacked: permutations differ");
        }
        int ndev = 0;
        ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
        if (ndev == 0) throw CudaError("CUDA: no device");
        DevGuard dg(o.device);
        auto L = std::make_unique<spqr_layer>();
        ck(cudaGetDevice(&L->device), "cudaGetDevice");
        L->stacked = true;
        L->prefix.assign(streams[0], streams[0] + v0.rec_off);
        L->geo = spqr::detail::geometry_from_prefix(L->prefix.data(), L->prefix.size());
        std::memset(&L->info, 0, sizeof(L->info));
        L->info.cols = v0.cols; L->info.weight_bits = v0.wb; L->info.scale_bits = v0.sb; L->info.zero_bits = v0.zb;
        L->info.beta1 = v0.b1; L->info.beta2 = v0.b2; L->info.flags = v0.flags;
        L->info.has_permutation = v0.has_permutation; L->info.tau = v0.tau; L->info.lambda_rel = v0.lambda_rel;
        L->info.device = L->device;
        for (int i = 0; i < count; ++i) {
            L->info.rows += views[i].rows;
            L->info.outlier_count += views[i].nnz;
            L->info.payload_bytes += sizes[i] - spqr::kSpqrHeaderBytes;
        }
        std::uint64_t dev_bytes = 0;
        if (v0.has_permutation) {
            std::vector<std::uint32_t> ord(v0.cols);
            for (std::uint32_t k = 0; k < v0.cols; ++k) ord[k] = v0.order(k);
            L->d_order = dalloc<std::uint32_t>(v0.cols);
            ck(cudaMemcpy(L->d_order, ord.data(), 4ull * v0.cols, cudaMemcpyHostToDevice), "H2D order");
            dev_bytes += 4ull * v0.cols;
        }
        L->fast = true;
        if (o.host_transcode) {
            spqr::detail::TiledHost t;
            for (int i = 0; i < count; ++i) {
                const spqr::detail::TiledHost ti = spqr::detail::transcode_to_tiled(views[i], 0);
                const std::uint64_t base = t.cells.size();
                if (base + ti.cells.size() > 0xfffffff0ull) spqr::fail(spqr::Errc::config_invalid, "stacked: too large");
                if (i == 0) {
                    t.Pn = ti.Pn;
                    t.cell_bytes = ti.cell_bytes;
                    t.prefix = ti.prefix;
                }
                t.Gn += ti.Gn;
                t.cells.insert(t.cells.end(), ti.cells.begin(), ti.cells.end());
                if (!t.cell_off.empty()) t.cell_off.pop_back();
                for (std::uint32_t off : ti.cell_off) t.cell_off.push_back(static_cast<std::uint32_t>(base + off));
            }
            dev_bytes += upload_tiled(L.get(), t, views);
        } else {  // members' streams visit the device only for the transcode
            std::vector<std::uint8_t*> tmp;
            std::vector<const std::uint8_t*> dv;
            try {
                for (int i = 0; i < count; ++i) {
                    tmp.push_back(dalloc<std::uint8_t>(sizes[i] + 16));
                    ck(cudaMemcpy(tmp.back(), streams[i], sizes[i], cudaMemcpyHostToDevice), "H2D member stream");
                    dv.push_back(tmp.back());
                }
                dev_bytes += transcode_on_device(L.get(), views, dv);
            } catch (...) {
                for (auto* q : tmp) cudaFree(q);
                throw;
            }
            for (auto* q : tmp) cudaFree(q);
        }
        L->info.fast_path = 1;
        ensure_own_ws(L.get(), 1);
        dev_bytes += L->ws_bytes;
        L->info.device_bytes = dev_bytes;
        *out = L.release();
    });
}

void spqr_layer_destroy(spqr_layer* layer) {
    if (!layer) return;
    DevGuard dg(layer->device);
    delete layer;
}

int spqr_layer_get_info(const spqr_layer* layer, spqr_layer_info* info) {
    return guard([&] { *info = layer->info; });
}

int spqr_layer_set_exact(spqr_layer* L, int exact) {
    return guard([&] {
        DevGuard dg(L->device);
        std::lock_guard<std::mutex> lk(L->mu);
        L->exact = exact != 0;
        if (L->hgraph) cudaGraphExecDestroy(L->hgraph);  // the host API's graph bakes the path in
        L->hgraph = nullptr;
    });
}

int spqr_layer_export_stream(const spqr_layer* L, uint8_t* out, size_t cap, size_t* len) {
    int rc = SPQR_OK;
    const int g = guard([&] {
        if (L->stacked) spqr::fail(spqr::Errc::config_invalid, "export of a stacked layer handle");
        DevGuard dg(L->device);
        std::vector<std::uint8_t> bytes;
        if (L->fast) {
            spqr::detail::TiledHost t;
            t.Gn = L->Gn; t.Pn = L->Pn; t.cell_bytes = L->cell_bytes; t.prefix = L->prefix;
            t.cell_off.resize(static_cast<std::size_t>(t.Gn) * t.Pn + 1);
            ck(cudaMemcpy(t.cell_off.data(), L->d_cell_off, 4 * t.cell_off.size(), cudaMemcpyDeviceToHost),
               "D2H cell_off");
            t.cells.resize(t.cell_off.back());
            ck(cudaMemcpy(t.cells.data(), L->d_cells, t.cells.size(), cudaMemcpyDeviceToHost), "D2H cells");
            bytes = spqr::detail::tiled_to_stream(L->geo, t, 0);
        } else {
            bytes.resize(L->info.payload_bytes + spqr::kSpqrHeaderBytes);
            ck(cudaMemcpy(bytes.data(), L->d_stream, bytes.size(), cudaMemcpyDeviceToHost), "D2H stream");
        }
        *len = bytes.size();
        if (!out || cap < bytes.size()) {
            spqr::detail::set_last_error("buffer too small");
            rc = SPQR_E_BUFFER_TOO_SMALL;
            return;
        }
        std::memcpy(out, bytes.data(), bytes.size());
    });
    return g ? g : rc;
}

int spqr_dequantize(const spqr_layer* L, float* w_dev, void* cuda_stream) {
    return guard([&] {
        if (L->stacked) spqr::fail(spqr::Errc::config_invalid, "dequantize of a stacked layer handle");
        DevGuard dg(L->device);
        auto st = static_cast<cudaStream_t>(cuda_stream);
        g_launches = 0;
        if (L->fast) {  // straight from the cell records (no raw stream in HBM)
            const unsigned blocks = static_cast<unsigned>((2ull * L->Gn * L->Pn * 32 + 255) / 256);
            const std::uint32_t m = L->info.rows, n = L->info.cols;
            auto run = [&](auto kern) {
                kern<<<blocks, 256, 0, st>>>(L->d_cells, L->d_cell_off, L->Gn, L->Pn, m, n, L->d_order, w_dev);
            };
            switch (L->info.weight_bits * 10 + L->info.scale_bits) {
                case 22: run(spqr_dev::dequant_cells<2, 2>); break;
                case 23: run(spqr_dev::dequant_cells<2, 3>); break;
                case 24: run(spqr_dev::dequant_cells<2, 4>); break;
                case 32: run(spqr_dev::dequant_cells<3, 2>); break;
                case 33: run(spqr_dev::dequant_cells<3, 3>); break;
                case 34: run(spqr_dev::dequant_cells<3, 4>); break;
                case 42: run(spqr_dev::dequant_cells<4, 2>); break;
                case 43: run(spqr_dev::dequant_cells<4, 3>); break;
                default: run(spqr_dev::dequant_cells<4, 4>); break;
            }
            ck(cudaGetLastError(), "launch dequant_cells");
            g_launches = 1;
            return;
        }
        const spqr_dev::RawGeom geo = raw_geom(L);
        const std::uint64_t total = static_cast<std::uint64_t>(geo.rows) * geo.nblocks;
        const unsigned blocks = static_cast<unsigned>(std::min<std::uint64_t>((total + 255) / 256, 1u << 20));
        spqr_dev::dequant_raw<<<blocks, 256, 0, st>>>(geo, w_dev);
        ck(cudaGetLastError(), "launch dequant_raw");
        spqr_dev::outliers_raw<<<(geo.rows + 255) / 256, 256, 0, st>>>(geo, w_dev);
        ck(cudaGetLastError(), "launch outliers_raw");
        g_launches = 2;
    });
}

uint64_t spqr_workspace_bytes(const spqr_layer* L, int batch) { return ws_layout(L, batch).total; }

int spqr_matvec_ws(const spqr_layer* L, const void* x_dev, int x_dtype, float* y_dev, int batch, void* ws,
                   uint64_t ws_bytes, void* cuda_stream) {
    return guard([&] {
        DevGuard dg(L->device);
        g_launches = 0;
        run_matvec(L, x_dev, x_dtype, y_dev, batch, ws, ws_bytes, static_cast<cudaStream_t>(cuda_stream));
    });
}

int spqr_matvec(const spqr_layer* L, const void* x_dev, int x_dtype, float* y_dev, int batch, void* cuda_stream) {
    return guard([&] {
        DevGuard dg(L->device);
        g_launches = 0;
        std::lock_guard<std::mutex> lk(L->mu);
        ensure_own_ws(L, batch);
        run_matvec(L, x_dev, x_dtype, y_dev, batch, L->d_ws, L->ws_bytes, static_cast<cudaStream_t>(cuda_stream));
    });
}

int spqr_gather_create(int device, uint32_t rows, int world, int rank, spqr_gather** out) {
    *out = nullptr;
    return guard([&] {
        if (world < 1 || world > spqr_dev::kMaxPeers + 1 || rank < 0 || rank >= world)
            spqr::fail(spqr::Errc::config_invalid, "gather: world must be 1..8 and 0 <= rank < world");
        DevGuard dg(device);
        auto g = std::make_unique<spqr_gather>();
        g->device = device; g->world = world; g->rank = rank; g->rows = rows;
        ck(cudaMalloc(&g->base, spqr_gather::kY + 4ull * rows), "cudaMalloc(gather)");
        ck(cudaMemset(g->base, 0, spqr_gather::kY + 4ull * rows), "memset(gather)");
        g->peer[rank] = g->base;
        *out = g.release();
    });
}

int spqr_gather_handle(const spqr_gather* g, void* out) {
    return guard([&] {
        static_assert(sizeof(cudaIpcMemHandle_t) == SPQR_GATHER_HANDLE_BYTES, "IPC handle size");
        DevGuard dg(g->device);
        cudaIpcMemHandle_t h;
        ck(cudaIpcGetMemHandle(&h, g->base), "cudaIpcGetMemHandle");
        std::memcpy(out, &h, sizeof h);
    });
}

int spqr_gather_open(spqr_gather* g, const void* handles, const uint32_t* row_base) {
    return guard([&] {
        DevGuard dg(g->device);
        if (g->open) spqr::fail(spqr::Errc::config_invalid, "gather: already open");
        const auto* hb = static_cast<const std::uint8_t*>(handles);
        for (int j = 0; j < g->world; ++j) {
            g->row_base[j] = row_base[j];
            if (j == g->rank) continue;
            cudaIpcMemHandle_t h;
            std::memcpy(&h, hb + static_cast<std::size_t>(j) * SPQR_GATHER_HANDLE_BYTES, sizeof h);
            void* ptr = nullptr;
            ck(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
            g->peer[j] = static_cast<std::uint8_t*>(ptr);
        }
        g->open = true;
    });
}

float* spqr_gather_y(const spqr_gather* g) { return g ? g->y() : nullptr; }

int spqr_matvec_gather(const spqr_layer* L, const void* x_dev, int x_dtype, spqr_gather* g, void* cuda_stream) {
    return guard([&] {
        DevGuard dg(L->device);
        g_launches = 0;
        if (!g->open) spqr::fail(spqr::Errc::config_invalid, "gather: spqr_gather_open first");
        if (g->device != L->device) spqr::fail(spqr::Errc::config_invalid, "gather: layer and buffer devices differ");
        if (!L->fast)
            spqr::fail(spqr::Errc::config_invalid, "fused all-gather needs a fast-path (tiled) layer");
        if (x_dtype != SPQR_F16 && x_dtype != SPQR_F32) spqr::fail(spqr::Errc::config_invalid, "x dtype must be f16 or f32");
        const std::uint32_t rb = g->row_base[g->rank];
        if (rb + L->info.rows > g->rows) spqr::fail(spqr::Errc::shape_mismatch, "gather: band beyond the full y");
        std::lock_guard<std::mutex> lk(L->mu);
        ensure_own_ws(L, 1);
        const WsLayout w = ws_layout(L, 1);
        const int f16 = x_dtype == SPQR_F16;
        spqr_dev::CtaParams p = cta_params(L, x_dev, f16 ? 0 : 1, g->y() + rb, static_cast<std::uint8_t*>(L->d_ws), w);
        std::uint32_t k = 0;
        for (int j = 0; j < g->world; ++j) {
            if (j != g->rank) p.ypeer[k++] = reinterpret_cast<float*>(g->peer[j] + spqr_gather::kY);
            p.pflags[j] = reinterpret_cast<std::uint32_t*>(g->peer[j]);
        }
        p.npeer = k;
        p.nflag = static_cast<std::uint32_t>(g->world);
        p.row_base = rb;
        p.rank = static_cast<std::uint32_t>(g->rank);
        p.done_ctr = reinterpret_cast<std::uint32_t*>(g->base + 68);
        p.round = reinterpret_cast<const std::uint32_t*>(g->base + 64);
        p.started = reinterpret_cast<const std::uint32_t*>(g->base + 4 * spqr_dev::kGatherStartedWord);
        const auto& c = L->cta[f16 ? 0 : 1];
        ck(spqr_dev::launch_cta_gather(static_cast<int>(L->info.weight_bits), static_cast<int>(L->info.scale_bits), !f16,
                                       c.shared_x, p, c.grid, c.smem, kNC, kSmemLimit,
                                       static_cast<cudaStream_t>(cuda_stream)),
           "launch gemv_cta (fused all-gather)");
        ++g_launches;
    });
}

int spqr_gather_wait(spqr_gather* g, void* cuda_stream) {
    // the wait is fused into the band kernel's last CTA (gemv_cta GATHER):
    // the stream is already ordered after every rank's rows of the round
    (void)g;
    (void)cuda_stream;
    g_launches = 0;
    return SPQR_OK;
}

void spqr_gather_destroy(spqr_gather* g) {
    if (!g) return;
    DevGuard dg(g->device);
    delete g;
}

int spqr_matvec_stage(const spqr_layer* L, const void* x_dev, int x_dtype, float* y_dev, int batch, int stage,
                      void* cuda_stream) {
    return guard([&] {
        DevGuard dg(L->device);
        g_launches = 0;
        if (stage < 0 || stage > 2) spqr::fail(spqr::Errc::config_invalid, "stage must be 0, 1 or 2");
        std::lock_guard<std::mutex> lk(L->mu);
        ensure_own_ws(L, batch);
        run_matvec(L, x_dev, x_dtype, y_dev, batch, L->d_ws, L->ws_bytes, static_cast<cudaStream_t>(cuda_stream),
                   stage);
    });
}

int spqr_matvec_host(const spqr_layer* L, const float* x_host, float* y_host, int batch) {
    return guard([&] {
        DevGuard dg(L->device);
        g_launches = 0;
        std::lock_guard<std::mutex> lk(L->mu);
        if (batch < 1) spqr::fail(spqr::Errc::shape_mismatch, "batch must be >= 1");
        if (L->wsh_bytes < ws_layout(L, batch).total) {  // the graph bakes the workspace in
            if (L->hgraph) cudaGraphExecDestroy(L->hgraph);
            L->hgraph = nullptr;
            ensure_ws(L, batch, L->d_wsh, L->wsh_bytes);
        }
        const std::size_t nx = static_cast<std::size_t>(L->info.cols) * batch;
        const std::size_t ny = static_cast<std::size_t>(L->info.rows) * batch;
        if (L->xh_cap < nx || L->yh_cap < ny) {  // device and pinned staging, grown together
            if (L->hgraph) cudaGraphExecDestroy(L->hgraph);
            L->hgraph = nullptr;
            for (float** d : {&L->d_xh, &L->d_yh})
                if (*d) cudaFree(*d);
            for (float** h : {&L->h_x, &L->h_y})
                if (*h) cudaFreeHost(*h);
            L->d_xh = L->d_yh = L->h_x = L->h_y = nullptr;
            L->xh_cap = std::max(L->xh_cap, nx);
            L->yh_cap = std::max(L->yh_cap, ny);
            L->d_xh = dalloc<float>(L->xh_cap);
            L->d_yh = dalloc<float>(L->yh_cap);
            ck(cudaHostAlloc(&L->h_x, 4 * L->xh_cap, cudaHostAllocDefault), "cudaHostAlloc(x staging)");
            ck(cudaHostAlloc(&L->h_y, 4 * L->yh_cap, cudaHostAllocDefault), "cudaHostAlloc(y staging)");
        }
        if (!L->hst) {
            ck(cudaStreamCreateWithFlags(&L->hst, cudaStreamNonBlocking), "stream (host API)");
            ck(cudaHostAlloc(&L->h_flag, 64, cudaHostAllocDefault), "cudaHostAlloc(flag)");
            *reinterpret_cast<volatile std::uint32_t*>(L->h_flag) = 0u;
            L->d_seq = dalloc<std::uint32_t>(1);
            ck(cudaMemset(L->d_seq, 0, 4), "memset seq");
            L->h_seq = 0;
        }
        // caller buffers that are page-locked are read / written directly by
        // the kernels; pageable ones go through the pinned staging.  The kind
        // is looked up once per pointer (the same buffers come back call after
        // call in a decode loop)
        auto pinned = [&](int k, const void* ptr) {
            if (L->pk_ptr[k] == ptr) return L->pk_pinned[k];
            cudaPointerAttributes a{};
            bool pin = false;
            if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess)
                cudaGetLastError();
            else
                pin = a.type == cudaMemoryTypeHost;
            L->pk_ptr[k] = ptr;
            L->pk_pinned[k] = pin;
            return pin;
        };
        const bool px = pinned(0, x_host), py = pinned(1, y_host);
        const void* src = px ? static_cast<const void*>(x_host) : L->h_x;
        void* dst = py ? static_cast<void*>(y_host) : L->h_y;
        if (!px) std::memcpy(L->h_x, x_host, 4 * nx);
        if (!L->hgraph || L->hg_batch != batch || L->hg_src != src || L->hg_dst != dst) {
            if (L->hgraph) cudaGraphExecDestroy(L->hgraph);
            L->hgraph = nullptr;
            cudaGraph_t g = nullptr;
            ck(cudaStreamBeginCapture(L->hst, cudaStreamCaptureModeThreadLocal), "capture (host API)");
            try {
                // x: a copy kernel reads the page-locked host vector over the
                // bus (UVA); y: the kernels store straight into page-locked
                // host memory (posted writes, flushed by kernel completion)
                if ((nx & 3u) == 0 && (reinterpret_cast<std::uintptr_t>(src) & 15u) == 0) {
                    const std::uint32_t n16 = static_cast<std::uint32_t>(nx / 4);
                    spqr_dev::copy_in<<<std::min<std::uint32_t>((n16 + 255) / 256, 64), 256, 0, L->hst>>>(
                        static_cast<const uint4*>(src), reinterpret_cast<uint4*>(L->d_xh), n16);
                    ck(cudaGetLastError(), "launch copy_in");
                    ++g_launches;
                } else {
                    ck(cudaMemcpyAsync(L->d_xh, src, 4 * nx, cudaMemcpyHostToDevice, L->hst), "H2D x");
                }
                run_matvec(L, L->d_xh, SPQR_F32, static_cast<float*>(dst), batch, L->d_wsh, L->wsh_bytes, L->hst);
                {
                    cudaLaunchConfig_t cfg{};
                    cfg.gridDim = dim3(1);
                    cfg.blockDim = dim3(1);
                    cfg.stream = L->hst;
                    cudaLaunchAttribute attr[1];
                    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                    attr[0].val.programmaticStreamSerializationAllowed = 1;
                    cfg.attrs = attr;
                    cfg.numAttrs = 1;
                    ck(cudaLaunchKernelEx(&cfg, spqr_dev::signal_host, L->d_seq,
                                          static_cast<volatile std::uint32_t*>(L->h_flag)),
                       "launch signal_host");
                }
            } catch (...) {
                cudaStreamEndCapture(L->hst, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            ck(cudaStreamEndCapture(L->hst, &g), "end capture (host API)");
            const cudaError_t e = cudaGraphInstantiate(&L->hgraph, g, 0);
            cudaGraphDestroy(g);
            ck(e, "instantiate (host API)");
            L->hg_batch = batch;
            L->hg_src = src;
            L->hg_dst = dst;
            L->hg_launches = g_launches + 1;  // + signal_host
        }
        ck(cudaGraphLaunch(L->hgraph, L->hst), "graph launch (host API)");
        // completion: spin on the page-locked word the graph's last node
        // posts (~1 us after the kernels) instead of a stream synchronisation
        // (~10 us); the stream is polled now and then so a failed launch
        // surfaces as an error instead of a hang
        const std::uint32_t want = ++L->h_seq;
        const volatile std::uint32_t* flag = L->h_flag;
        for (std::uint32_t it = 1; *flag != want; ++it) {
            if ((it & 4095u) == 0u) {
                const cudaError_t e = cudaStreamQuery(L->hst);
                if (e == cudaSuccess && *flag != want) {  // graph done but no signal: resync the sequence
                    ck(cudaMemcpy(&L->h_seq, L->d_seq, 4, cudaMemcpyDeviceToHost), "seq readback");
                    break;
                }
                if (e != cudaSuccess && e != cudaErrorNotReady) ck(e, "host-API graph");
            }
#if defined(__x86_64__)
            __builtin_ia32_pause();
#endif
        }
        g_launches = L->hg_launches;
        if (!py) std::memcpy(y_host, L->h_y, 4 * ny);
    });
}

int spqr_dense_gemv_f16(const void* w_dev, const void* x_dev, float* y_dev, uint32_t rows, uint32_t cols,
                        void* cuda_stream) {
    return guard([&] {
        g_launches = 0;
        int sms = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const unsigned grid = std::min<unsigned>((rows + 7) / 8, static_cast<unsigned>(sms) * 8);
        spqr_dev::dense_gemv_f16<<<grid, 256, 0, static_cast<cudaStream_t>(cuda_stream)>>>(
            static_cast<const __half*>(w_dev), static_cast<const __half*>(x_dev), y_dev, rows, cols);
        ck(cudaGetLastError(), "launch dense_gemv_f16");
        g_launches = 1;
    });
}

int spqr_last_launch_count(void) { return g_launches; }

int spqr_debug_layer_cells(const spqr_layer* L, uint8_t* cells, size_t cap, size_t* len, uint32_t* cell_off) {
    return guard([&] {
        if (!L->fast) spqr::fail(spqr::Errc::config_invalid, "not a tiled layer");
        DevGuard dg(L->device);
        const std::size_t ncell = static_cast<std::size_t>(L->Gn) * L->Pn;
        std::vector<std::uint32_t> off(ncell + 1);
        ck(cudaMemcpy(off.data(), L->d_cell_off, 4 * off.size(), cudaMemcpyDeviceToHost), "D2H cell_off");
        *len = off.back();
        if (cell_off) std::memcpy(cell_off, off.data(), 4 * off.size());
        if (cells && cap >= off.back())
            ck(cudaMemcpy(cells, L->d_cells, off.back(), cudaMemcpyDeviceToHost), "D2H cells");
    });
}

#ifdef SPQR_TIMELINE
// tools-only: copy the gemv_tiled per-warp timeline (8 x u64 per warp)
int spqr_debug_timeline(unsigned long long* host, size_t count) {
    return guard([&] {
        ck(cudaMemcpyFromSymbol(host, spqr_dev::g_timeline, 8 * std::min<size_t>(count, 148 * 32 * 8)),
           "timeline");
    });
}
#endif

int spqr_bench_layer(const spqr_layer* L, int repeats, double* ns3) {
    return guard([&] {
        if (repeats < 1) spqr::fail(spqr::Errc::config_invalid, "repeats must be >= 1");
        DevGuard dg(L->device);
        const std::size_t m = L->info.rows, n = L->info.cols;
        float* x = dalloc<float>(n);
        float* y = dalloc<float>(m);
        float* w = dalloc<float>(m * n);
        __half* w16 = dalloc<__half>(m * n);
        __half* x16 = dalloc<__half>(n);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        auto cleanup = [&] {
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
            cudaFree(x); cudaFree(y); cudaFree(w); cudaFree(w16); cudaFree(x16);
        };
        try {
            ck(cudaMemset(x, 0, 4 * n), "memset");
            ck(cudaMemset(w16, 0, 2 * m * n), "memset");
            ck(cudaMemset(x16, 0, 2 * n), "memset");
            ensure_own_ws(L, 1);
            auto time_it = [&](auto&& body) {
                body();  // warm-up
                std::vector<float> ms(repeats);
                for (int i = 0; i < repeats; ++i) {
                    cudaEventRecord(e0, nullptr);
                    body();
                    cudaEventRecord(e1, nullptr);
                    ck(cudaEventSynchronize(e1), "event sync");
                    cudaEventElapsedTime(&ms[i], e0, e1);
                }
                std::sort(ms.begin(), ms.end());
                const int mid = repeats / 2;
                return 1e6 * (repeats % 2 ? ms[mid] : 0.5 * (ms[mid - 1] + ms[mid]));
            };
            ns3[0] = time_it([&] { run_matvec(L, x, SPQR_F32, y, 1, L->d_ws, L->ws_bytes, nullptr); });
            ns3[1] = time_it([&] { spqr_dequantize(L, w, nullptr); });
            int sms = 0;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, L->device);
            const unsigned grid = std::min<unsigned>((m + 7) / 8, static_cast<unsigned>(sms) * 8);
            ns3[2] = time_it([&] {
                spqr_dev::dense_gemv_f16<<<grid, 256>>>(w16, x16, y, static_cast<std::uint32_t>(m),
                                                        static_cast<std::uint32_t>(n));
            });
            ck(cudaGetLastError(), "bench launches");
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
    });
}

int spqr_dev_alloc(void** ptr, size_t bytes) {
    return guard([&] { ck(cudaMalloc(ptr, bytes ? bytes : 1), "cudaMalloc"); });
}
void spqr_dev_free(void* ptr) {
    if (ptr) cudaFree(ptr);
}
int spqr_dev_copy_to_host(void* dst, const void* src, size_t bytes) {
    return guard([&] { ck(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost), "D2H"); });
}
int spqr_dev_copy_to_device(void* dst, const void* src, size_t bytes) {
    return guard([&] { ck(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice), "H2D"); });
}

}  // extern "C"
