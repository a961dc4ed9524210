// gemm_tc.cuh -- batched SpQR decode (batch >= 2): dequantize to fp16 in
// shared memory, then tcgen05.mma (sm_100a 5th-generation tensor cores, fp32
// accumulators in TMEM).  Included by kernels.cuh (namespace spqr_dev).
//
// Reference semantics: matvec(t, x, plan) (kernel.hpp:89-124) applied to each
// of the B batch columns; the weights are dequantize_full's (kernel.hpp:17-25,
// solver.hpp:345-362: s*(q - z), then + fp16 outlier), rounded once to fp16
// (scaled by 2^-sigma, an exact per-layer power of two that keeps every
// operand in fp16 range), which is what makes the product a dense
// contraction the tensor cores can run (BASELINE north star: "dequant-then-
// mma path for batch >= 16").  Accumulation is fp32 in TMEM; the tolerance is
// the north star's 1e-3 relative (fp16 weight rounding costs ~1e-4).
//
// Tiles: 128 rows (four 32-row cell rows) x 128 columns (half a 256-column
// panel) per MMA stage, N = batch padded to 16 (<= 64 per launch).
//   * 16 dequant warps (warp = 8 unit + 4 half + cell row; HPW = 2 folds the
//     two column halves into one warp): the first warp of each cell row streams
//     that row's cells (cp.async.bulk, two record slots, one cell of
//     lookahead, record offsets loaded a step ahead); each warp decodes the
//     bilevel statistics of its (unit, half) into a per-(row, block) fp16 table
//     {s 2^(-p-sigma) for both k halves, 1024 + round(z) 2^p, -s (z - round z)
//     2^-sigma}, turns every A-fragment register of codes (the batch-1 layout;
//     ONE LOP3 makes each half the binary16 normal 1024 + code*2^p, p <= 7)
//     into weights with one exact HSUB2 and ONE HFMA2 (sigma puts the largest
//     weights near 2^12, so small weights stay binary16 normals), and writes
//     them with stmatrix into the
//     UMMA K-major core-matrix layout; the four warps of a cell row then add the
//     cell's outliers in place between two named barriers; after a tile's last
//     stage the warps whose TMEM lane quarter holds the rows read the
//     accumulator back (tcgen05.ld) and write y;
//   * the control warp: allocates TMEM (two accumulators of N columns), copies
//     each stage's x tile (prepared by xprep_tc in the same layout), issues the
//     8 tcgen05.mma of a stage and commits them to mbarriers.
// A stages are 3- or 4-buffered (by shared memory), x tiles 3-buffered;
// accumulators are double-buffered across 128-row tiles so the epilogue of one
// tile overlaps the next tile's MMAs.  Split-K across CTAs: each CTA owns a
// contiguous, byte-balanced range of (tile, panel) units; partial tiles go
// through partial slots and a per-warp acq_rel counter, the last contributor
// adding them in range order.

struct TcParams {
    const std::uint8_t* cells;        // cell records (batch-1 layout)
    const std::uint32_t* cell_off;    // [ncell+1]
    const std::uint32_t* cta_start;   // [nv+1] first unit (T * Pn + P) of each range
    const std::uint32_t* gmap;        // [Tn][2] {partial slot base, contributing ranges}
    const std::uint32_t* cmap;        // [nv][2] ordinal of the range in its first / last tile
    const std::uint8_t* xpanels;      // [2*Pn][N x 128 fp16] x tiles (xprep_tc)
    float* y;                         // [B][m]
    float* partial;                   // [slots][N][128]
    std::uint32_t* counters;          // [Tn][16] (per dequant warp), zero between launches
    std::uint32_t m, Pn, Gn, Tn, nv, B, N;
    std::uint32_t rec_cap, slot_bytes;
    std::uint32_t pn_magic;           // u / Pn == umulhi(u, pn_magic) (Pn > 1)
    float out_scale;                  // 2^sigma
    int sigma;
    std::uint32_t na;                 // A stage buffers (3 or 4, by shared memory)
    std::uint32_t Nh;                 // fp32 x: lo parts in accumulator columns Nh .. 2Nh-1 (0: fp16 x)
};

namespace tc {
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ std::uint64_t smem_desc(std::uint32_t addr, std::uint32_t lbo, std::uint32_t sbo) {
    // K-major, no swizzle: core matrices of 8 rows x 16 B; lbo = stride between
    // the two K core matrices of an MMA, sbo = stride between 8-row groups
    return static_cast<std::uint64_t>((addr >> 4) & 0x3FFFu) |
           (static_cast<std::uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
           (static_cast<std::uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);  // version 1 (sm_100)
}
__device__ __forceinline__ void mma_f16(std::uint32_t d_tmem, std::uint64_t a, std::uint64_t b, std::uint32_t idesc,
                                        std::uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
        : "memory");
}
// issued by a whole warp (warp-uniform operands stay in uniform registers: ~20
// cycles per small MMA instead of ~60 from a lone lane, tools/umma_bench.cu);
// one elected lane issues
__device__ __forceinline__ void mma_f16_e(std::uint32_t d_tmem, std::uint64_t a, std::uint64_t b, std::uint32_t idesc,
                                          std::uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
        : "memory");
}
// One stage of the control warp: 8 MMAs along K (16 columns each) issued by
// one elected lane, the descriptors' start-address words stepped by ainc /
// binc (16-B units; the 14-bit address field never carries for shared memory),
// then the commits to the two buffer-free barriers -- one elect for the lot
__device__ __forceinline__ void mma8_f16_e(std::uint32_t d_tmem, std::uint64_t a, std::uint64_t b, std::uint32_t ainc,
                                           std::uint32_t binc, std::uint32_t idesc, std::uint32_t accumulate,
                                           std::uint32_t bar0, std::uint32_t bar1) {
    const std::uint32_t alo = static_cast<std::uint32_t>(a), ahi = static_cast<std::uint32_t>(a >> 32);
    const std::uint32_t blo = static_cast<std::uint32_t>(b), bhi = static_cast<std::uint32_t>(b >> 32);
#define SPQR_MMA8_STEP                                                                 \
    "add.u32 al, al, %7;\n\tadd.u32 bl, bl, %8;\n\tmov.b64 a, {al, %2};\n\tmov.b64 b, {bl, %4};\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, t;\n\t"
    asm volatile(
        "{\n\t.reg .pred p, e, t;\n\t.reg .b32 al, bl;\n\t.reg .b64 a, b;\n\t"
        "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %6, 0;\n\tsetp.eq.b32 t, %6, %6;\n\t"
        "mov.b32 al, %1;\n\tmov.b32 bl, %3;\n\tmov.b64 a, {al, %2};\n\tmov.b64 b, {bl, %4};\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, p;\n\t"
        SPQR_MMA8_STEP SPQR_MMA8_STEP SPQR_MMA8_STEP SPQR_MMA8_STEP SPQR_MMA8_STEP SPQR_MMA8_STEP SPQR_MMA8_STEP
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%9];\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%10];\n\t}" ::"r"(d_tmem),
        "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc), "r"(accumulate), "r"(ainc), "r"(binc), "r"(bar0), "r"(bar1)
        : "memory");
#undef SPQR_MMA8_STEP
}
__device__ __forceinline__ void commit_e(std::uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void commit(std::uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void ld16(std::uint32_t taddr, float (&v)[16]) {
    std::uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void stsm_x4(std::uint32_t addr, std::uint32_t a0, std::uint32_t a1, std::uint32_t a2,
                                        std::uint32_t a3) {
    // no "memory" clobber: the A stage is only read by the tensor core after the
    // (volatile, clobbering) proxy fence + mbarrier arrive, which stay ordered
    // after this volatile asm; the table loads may be scheduled across it
    asm volatile("stmatrix.sync.aligned.m8n8.x4.shared.b16 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(a0), "r"(a1),
                 "r"(a2), "r"(a3));
}
// (w & M) | bias in ONE LOP3 (the mask an immediate, the bias in a register;
// written as a plain C++ expression the compiler emits two)
template <std::uint32_t M>
__device__ __forceinline__ std::uint32_t and_or(std::uint32_t a, std::uint32_t c) {
    std::uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "n"(M), "r"(c));
    return d;
}
// the code pair at bit offset pb of a window as binary16 normals 1024 + q 2^pb
// (pb is a constant after unrolling, so the switch folds away)
template <std::uint32_t MASK>
__device__ __forceinline__ std::uint32_t code_bias(std::uint32_t win, int pb, std::uint32_t bias) {
    switch (pb) {
        case 0: return and_or<(MASK << 0) * 0x00010001u>(win, bias);
        case 1: return and_or<(MASK << 1) * 0x00010001u>(win, bias);
        case 2: return and_or<(MASK << 2) * 0x00010001u>(win, bias);
        case 3: return and_or<(MASK << 3) * 0x00010001u>(win, bias);
        case 4: return and_or<(MASK << 4) * 0x00010001u>(win, bias);
        case 5: return and_or<(MASK << 5) * 0x00010001u>(win, bias);
        case 6: return and_or<(MASK << 6) * 0x00010001u>(win, bias);
        default: return and_or<(MASK << 7) * 0x00010001u>(win, bias);
    }
}
// (a - (z, z)) * (s, s) + (c, c) per f16 lane; z, s, c are the low (HI=false)
// or high (HI=true) halves of their registers.  a - z is exact (1024 + q 2^p
// minus 1024 + round(z) 2^p, |round(z)| <= 15), so the weight is rounded once.
template <bool HI>
__device__ __forceinline__ std::uint32_t deq2(std::uint32_t a, std::uint32_t z, std::uint32_t s, std::uint32_t c) {
    std::uint32_t d;
    if constexpr (HI)
        asm("{\n\t.reg .b16 zl, zh, sl, sh, cl, ch;\n\t.reg .b32 z2, s2, c2, t;\n\t"
            "mov.b32 {zl, zh}, %2;\n\tmov.b32 z2, {zh, zh};\n\t"
            "mov.b32 {sl, sh}, %3;\n\tmov.b32 s2, {sh, sh};\n\t"
            "mov.b32 {cl, ch}, %4;\n\tmov.b32 c2, {cl, cl};\n\t"
            "sub.rn.f16x2 t, %1, z2;\n\tfma.rn.f16x2 %0, t, s2, c2;\n\t}"
            : "=r"(d)
            : "r"(a), "r"(z), "r"(s), "r"(c));
    else
        asm("{\n\t.reg .b16 zl, zh, sl, sh, cl, ch;\n\t.reg .b32 z2, s2, c2, t;\n\t"
            "mov.b32 {zl, zh}, %2;\n\tmov.b32 z2, {zl, zl};\n\t"
            "mov.b32 {sl, sh}, %3;\n\tmov.b32 s2, {sl, sl};\n\t"
            "mov.b32 {cl, ch}, %4;\n\tmov.b32 c2, {cl, cl};\n\t"
            "sub.rn.f16x2 t, %1, z2;\n\tfma.rn.f16x2 %0, t, s2, c2;\n\t}"
            : "=r"(d)
            : "r"(a), "r"(z), "r"(s), "r"(c));
    return d;
}
}  // namespace tc

// x tiles for the tensor cores: stage (P, h) holds columns 256P + 128h + k,
// k < 128, of every batch column n < N (zero for n >= B or beyond the layer)
// as fp16, K-major core matrices: byte (k/8)*16N + (n/8)*128 + (n%8)*16 + (k%8)*2.
// fp32 x (Nh > 0): columns nn < Nh carry fp16(x) of batch column nn, columns
// Nh + nn the residual fp16(x - fp16(x)); the epilogue adds the two
// accumulator columns, so x keeps ~22 significant bits on the tensor cores.
static __global__ void __launch_bounds__(256) xprep_tc(const void* __restrict__ x, int x_f16, std::uint32_t n,
                                                std::uint32_t B, std::uint32_t N, std::uint32_t Pn,
                                                const std::uint32_t* __restrict__ order, std::uint8_t* __restrict__ out,
                                                std::uint32_t Nh) {
    pdl_launch();
    const std::uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;  // (stage, n, k core)
    const std::uint32_t total = 2u * Pn * N * 16u;
    pdl_wait();
    if (idx >= total) return;
    const std::uint32_t kc = idx & 15u, nn = (idx >> 4) % N, st = idx / (16u * N);
    const std::uint32_t c0 = 128u * st + 8u * kc;  // st = 2P + h
    std::uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        float v2[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const std::uint32_t c = c0 + 2 * e + q;
            float v = 0.f;
            const bool lo = Nh && nn >= Nh;
            const std::uint32_t bc = lo ? nn - Nh : nn;  // batch column
            if (bc < B && c < n) {
                const std::uint32_t src = order ? __ldg(order + c) : c;
                const std::size_t off = static_cast<std::size_t>(bc) * n + src;
                v = x_f16 ? __half2float(static_cast<const __half*>(x)[off]) : static_cast<const float*>(x)[off];
                if (lo) v -= __half2float(__float2half_rn(v));
            }
            v2[q] = v;
        }
        w[e] = pack_h2_rn(v2[0], v2[1]);
    }
    std::uint8_t* dst = out + static_cast<std::size_t>(st) * 256u * N + kc * 16u * N + (nn >> 3) * 128u + (nn & 7u) * 16u;
    *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
}

// Dequant warps: each owns HPW column halves of one 16-row unit of one cell
// row, so 16 / HPW dequant warps + 1 control warp.  HPW = 1: 17 warps at 96
// registers (five share an SM sub-partition's 16K registers).  HPW = 2: 9
// warps, both halves interleaved in one warp -- 30 % fewer instructions
// (per-step bookkeeping and waits halve) at lower issue efficiency.  Measured
// on 8192x22016 (tools/batch_sweep.py): HPW = 2 is 2-4 % faster up to 32
// batch columns, HPW = 1 10 % faster at 64 -- the launch picks by N.
__host__ __device__ constexpr int tc_dequant_warps(int hpw) { return 16 / hpw; }
__host__ __device__ constexpr int tc_threads(int hpw) { return 32 * (16 / hpw + 1); }
__host__ __device__ constexpr std::uint32_t tc_tab_stride(int hpw) { return 16u * 8u * hpw + 16u; }  // 8 HPW blocks x 16 B + pad
__host__ __device__ constexpr std::uint32_t tc_tab_bytes(int hpw) {  // all warps' tables
    return static_cast<std::uint32_t>(16 / hpw) * 16u * tc_tab_stride(hpw);
}
constexpr std::uint32_t kTcTabBytes = tc_tab_bytes(1) > tc_tab_bytes(2) ? tc_tab_bytes(1) : tc_tab_bytes(2);
constexpr int kTcHpwMaxN = 32;  // HPW = 2 up to this many MMA columns, HPW = 1 above (N = 48: HPW = 1 5-10 % faster)
template <int BW, int BS, int BZ, int HPW>
__global__ void __launch_bounds__(tc_threads(HPW), 1) gemm_tc(const TcParams p) {
    using G = Geo<BW>;
    constexpr std::uint32_t UNIT = T::unit_bytes(BW, BS, BZ);
    constexpr std::uint32_t CELL = 2 * UNIT;
    constexpr std::uint32_t CODEB = T::code_bytes(BW);
    constexpr std::uint32_t STATB = T::stat_bytes(BS, BZ);
    constexpr std::uint32_t MASK = (1u << BW) - 1u;
    constexpr std::uint32_t SMASK = (1u << BS) - 1u, ZMASK = (1u << BZ) - 1u;
    constexpr float kMagic = 8388608.0f;
    constexpr std::uint32_t A_STAGE = 128u * 128u * 2u;  // 32 KB
    constexpr std::uint32_t KC_A = 2048u;                // A: bytes between k core matrices (16 row groups)
    constexpr int ND = tc_dequant_warps(HPW);           // dequant warps (HPW halves each)
    constexpr int RW = ND / 4;                           // dequant warps per cell row
    constexpr std::uint32_t TS = tc_tab_stride(HPW);
    constexpr int CTRL = ND;                             // control warp

    extern __shared__ __align__(128) std::uint8_t smem[];
    __shared__ std::uint64_t rec_full[4][2], rec_empty[4][2], a_full[4], a_free[4], b_full[3], b_free[3], d_full[2],
        d_free[2];
    __shared__ std::uint32_t slot_r[4][2][2];
    __shared__ std::uint32_t tmem_base;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const std::uint32_t N = p.N;
    const std::uint32_t B_STAGE = 256u * N;
#ifdef SPQR_TIMELINE
    unsigned long long tw[4] = {0, 0, 0, 0};
    const unsigned long long t_start = gtime();
#define TC_WAIT(i, expr)                      \
    {                                         \
        const unsigned long long t0_ = gtime(); \
        expr;                                 \
        tw[i] += gtime() - t0_;               \
    }
#else
#define TC_WAIT(i, expr) expr;
#endif
    const std::uint32_t tcols = N <= 16 ? 32u : (N <= 32 ? 64u : (N <= 64 ? 128u : 256u));
    const std::uint32_t NA = p.na;                              // A buffers (3 or 4)
    std::uint8_t* abuf = smem;                                  // [NA][A_STAGE]: stage s in buffer s % NA
    std::uint8_t* bbuf = smem + NA * A_STAGE;                   // [3][B_STAGE]: x tiles, 2 stages of lookahead
    std::uint8_t* recs = bbuf + 3 * B_STAGE;                    // [4 cell rows][2][slot_bytes]
    std::uint8_t* stab = recs + 8u * p.slot_bytes;              // [ND warps][16 rows][TS B: 8 HPW blocks x 16 B + pad]

    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i)
            for (int k = 0; k < 2; ++k) {
                mbar_init(&rec_full[i][k], 1);
                mbar_init(&rec_empty[i][k], RW);  // the dequant warps of the cell row
            }
        for (int b = 0; b < 4; ++b) {
            mbar_init(&a_full[b], 8);  // 4 cell rows x 2 units write a half stage
            mbar_init(&a_free[b], 1);
        }
        for (int b = 0; b < 3; ++b) {
            mbar_init(&b_full[b], 1);
            mbar_init(&b_free[b], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&d_full[b], 1);
            mbar_init(&d_free[b], ND);
        }
        fence_mbar_init();
    }
    // zero both A stages once: rows of missing row-group pairs (the layer's last
    // tile) then contribute 0 instead of whatever shared memory held
    for (std::uint32_t i = threadIdx.x; i < NA * A_STAGE / 16u; i += blockDim.x)
        reinterpret_cast<uint4*>(abuf)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async();
    if (warp == CTRL) {  // two accumulators of N fp32 columns each
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "r"(tcols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    pdl_launch();
    const std::uint32_t tmem = tmem_base;
    const std::uint32_t v = blockIdx.x;
    const std::uint32_t u0 = __ldg(p.cta_start + v), u1 = __ldg(p.cta_start + v + 1);
    const std::uint32_t nst = 2u * (u1 - u0);  // MMA stages of this range

    if (warp == CTRL) {
        // ------------------------------------------------------- control --
        // (the whole warp runs the loop: warp-uniform operands; elected lanes issue)
        {
            pdl_wait();  // xprep_tc has completed
            const std::uint32_t idesc = (1u << 4) | ((N >> 3) << 17) | ((128u >> 4) << 24);  // f16 x f16 -> f32, K-major
            auto pan = [&](std::uint32_t u) { return p.Pn == 1u ? 0u : u - __umulhi(u, p.pn_magic) * p.Pn; };
            auto issue_b = [&](std::uint32_t s) {  // x tile of stage s into buffer s % 3
                const std::uint32_t u = u0 + (s >> 1), P = pan(u);
                const std::uint32_t b = s % 3u;
                if (s >= 3) mbar_wait(&b_free[b], ((s / 3u) - 1u) & 1u);
                if (lane == 0) {
                    mbar_expect_tx(&b_full[b], B_STAGE);
                    bulk_g2s(bbuf + b * B_STAGE, p.xpanels + static_cast<std::size_t>(2u * P + (s & 1u)) * B_STAGE,
                             B_STAGE, &b_full[b]);
                }
                __syncwarp();
            };
            for (std::uint32_t s = 0; s < 2 && s < nst; ++s) issue_b(s);
            std::uint32_t tile_i = 0;  // tiles started in this range
            std::uint32_t b = 0, bn = 0;  // A buffer of stage s = s % NA, its use count s / NA
#pragma unroll 1
            for (std::uint32_t s = 0; s < nst; ++s) {
                const std::uint32_t u = u0 + (s >> 1), P = pan(u);
                const bool first = (s & 1u) == 0 && ((s >> 1) == 0 || P == 0);  // first stage of a tile
                const bool last = (s & 1u) && (u + 1 == u1 || P + 1 == p.Pn);
                if (first && tile_i >= 2) TC_WAIT(2, mbar_wait(&d_free[tile_i & 1u], ((tile_i >> 1) - 1u) & 1u))
                const std::uint32_t bb = s % 3u;
                TC_WAIT(0, mbar_wait(&a_full[b], bn & 1u))
                TC_WAIT(1, mbar_wait(&b_full[bb], (s / 3u) & 1u))
                tc::fence_after();
                const std::uint32_t d = tmem + (tile_i & 1u) * N;
                const std::uint32_t a_sa = smem_u32(abuf + b * A_STAGE), b_sa = smem_u32(bbuf + bb * B_STAGE);
                // A buffer b and x buffer bb are free once these MMAs finish
                tc::mma8_f16_e(d, tc::smem_desc(a_sa, KC_A, 128u), tc::smem_desc(b_sa, 16u * N, 128u),
                               2u * KC_A / 16u, 2u * N, idesc, first ? 0u : 1u, smem_u32(&a_free[b]),
                               smem_u32(&b_free[bb]));
                if (++b == NA) {
                    b = 0;
                    ++bn;
                }
                if (last) {
                    tc::commit_e(&d_full[tile_i & 1u]);
                    ++tile_i;
                }
                // x tile of stage s + 2 into the buffer of stage s - 1: its wait for
                // the MMAs of s - 1 comes after stage s is queued, so the tensor
                // pipe never drains between stages
                if (s + 2 < nst) issue_b(s + 2);
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------- dequant --
        // warp = 4 (HPW uu + hh) + ci (HPW = 1) or 4 uu + ci (HPW = 2): cell row
        // ci (row-group pair 4T + ci), unit uu (rows 16uu .. 16uu+15), column
        // half hh (blocks 8hh .. 8hh+7) or both; warp % 4 == ci, the TMEM lane
        // quarter the epilogue reads
        const int ci = warp & 3;
        const int uu = HPW == 2 ? warp >> 2 : warp >> 3;
        const int h0 = HPW == 2 ? 0 : (warp >> 2) & 1;  // first column half of this warp
        const int g = lane >> 2, t = lane & 3;
        std::uint8_t* ring = recs + static_cast<std::uint32_t>(ci) * 2u * p.slot_bytes;
        std::uint8_t* tab = stab + static_cast<std::uint32_t>(warp) * 16u * TS;  // 16 rows x TS B (padded: no bank conflicts)
        const std::uint32_t magic = 0x4B000000u;
        auto tile_of = [&](std::uint32_t u) { return p.Pn == 1u ? u : __umulhi(u, p.pn_magic); };
        auto cell_of = [&](std::uint32_t u, std::uint32_t& q) {
            const std::uint32_t T_ = tile_of(u), P = u - T_ * p.Pn;
            const std::uint32_t Gq = 4u * T_ + static_cast<std::uint32_t>(ci);
            q = Gq * p.Pn + P;
            return Gq < p.Gn;
        };
        // record k of this cell row goes to slot k & 1; warp ci (unit 0, half 0)
        // issues it once all warps of the row released the slot's previous
        // record.  The record offsets of unit u + 1 are loaded one step ahead
        // into (nr0, nr1), so the issuing lane never waits on a global load.
        std::uint32_t nr0 = 0, nr1 = 0;
        auto load_off = [&](std::uint32_t u) {
            std::uint32_t q;
            if (warp == ci && lane == 0 && u < u1 && cell_of(u, q)) {
                nr0 = __ldg(p.cell_off + q);
                nr1 = __ldg(p.cell_off + q + 1);
            }
        };
        auto issue = [&](std::uint32_t u, std::uint32_t k) {
            std::uint32_t q;
            if (warp == ci && lane == 0 && cell_of(u, q)) {
                const std::uint32_t sl = k & 1u;
                if (k >= 2) mbar_wait(&rec_empty[ci][sl], ((k >> 1) - 1u) & 1u);
                const std::uint32_t r0 = nr0, r1 = nr1;
                slot_r[ci][sl][0] = r0;
                slot_r[ci][sl][1] = r1;
                const std::uint32_t nb = min(r1 - r0, p.rec_cap);
                mbar_expect_tx(&rec_full[ci][sl], nb);
                bulk_g2s(ring + sl * p.slot_bytes, p.cells + r0, nb, &rec_full[ci][sl]);
            }
        };
        const float sig_scale = __uint_as_float(static_cast<std::uint32_t>(127 - p.sigma) << 23);  // 2^-sigma
        const std::uint32_t bias16 = 0x64006400u;  // binary16 1024 in both halves
        // per-lane constants of the statistics: blocks 8hh + 2t + bs, bs = 0, 1
        float2 f0, f1, g0, g1;  // s multipliers 2^(24-p-sigma) and code scales 2^(p-24), column halves 0 / 1
        {
            const int mm0 = (2 * t) % G::MPC, mm1 = (2 * t + 1) % G::MPC;
            auto pw = [](int e) { return __uint_as_float(static_cast<std::uint32_t>(127 + e) << 23); };
            f0 = make_float2(pw(-T::prescale_p(BW, 2 * mm0) - p.sigma), pw(-T::prescale_p(BW, 2 * mm1) - p.sigma));
            f1 = make_float2(pw(-T::prescale_p(BW, 2 * mm0 + 1) - p.sigma), pw(-T::prescale_p(BW, 2 * mm1 + 1) - p.sigma));
            g0 = make_float2(pw(T::prescale_p(BW, 2 * mm0)), pw(T::prescale_p(BW, 2 * mm1)));
            g1 = make_float2(pw(T::prescale_p(BW, 2 * mm0 + 1)), pw(T::prescale_p(BW, 2 * mm1 + 1)));
        }
        std::uint32_t k = 0;  // records of this cell row consumed so far
        load_off(u0);
        if (u0 < u1) issue(u0, 0);
        load_off(u0 + 1);
        pdl_wait();
        std::uint32_t tile_i = 0;
        std::uint32_t sb0 = 0, sn0 = 0;  // buffer / use count of stage 2it
        // stmatrix row address of this lane: matrix lane/8 = (row half, k half)
        const std::uint32_t mq = static_cast<std::uint32_t>(lane >> 3);
#pragma unroll 1
        for (std::uint32_t u = u0; u < u1; ++u) {
            std::uint32_t q;
            const bool have = cell_of(u, q);
            if (have && u + 1 < u1) {
                issue(u + 1, k + 1);
                load_off(u + 2);
            }
            const std::uint32_t sl = k & 1u;
            const std::uint8_t* cell = ring + sl * p.slot_bytes;
            const std::uint8_t* unit = cell + uu * UNIT;
            std::uint32_t r0 = 0, r1 = 0;
            if (have) {
                TC_WAIT(0, mbar_wait(&rec_full[ci][sl], (k >> 1) & 1u))
                r0 = slot_r[ci][sl][0];
                r1 = slot_r[ci][sl][1];
                // statistics: lane owns (row g + 8rho, block 8hh + 2t + bs) of unit uu
                // for this warp's halves hh; the two blocks bs = 0, 1 ride in the
                // halves of packed f32x2 math
                std::uint32_t st[2];  // lo (row g) / hi (row g + 8) statistic streams
                load_stat_streams<BS>(unit + CODEB, lane, st);
#pragma unroll
                for (int hi = 0; hi < HPW; ++hi) {
                    const int hh = h0 + hi;
                    const uint4 s4 = *reinterpret_cast<const uint4*>(unit + CODEB + STATB + (8 * hh + 2 * t) * 8);
                    const __half2 sh0 = u32_as_h2(s4.x), zh0 = u32_as_h2(s4.y), sh1 = u32_as_h2(s4.z),
                                  zh1 = u32_as_h2(s4.w);
                    const float2 Ss = make_float2(__low2float(sh0), __low2float(sh1));
                    const float2 Zs = make_float2(-__high2float(sh0), -__high2float(sh1));
                    const float2 Sz = make_float2(__low2float(zh0), __low2float(zh1));
                    const float2 Zz = make_float2(-__high2float(zh0), -__high2float(zh1));
#pragma unroll
                    for (int rho = 0; rho < 2; ++rho) {
                        // pairs j = 4 kind + 2 hh + bs at stream bit BS j (tiled.hpp)
                        const int j0 = T::stat_pair(0, hh, 0), j1 = T::stat_pair(0, hh, 1);
                        const float2 cs = fadd2(make_float2(magic_field_rt<SMASK>(st[rho], j0 * BS, magic),
                                                            magic_field_rt<SMASK>(st[rho], j1 * BS, magic)),
                                                make_float2(-kMagic, -kMagic));
                        const float2 cz = fadd2(make_float2(magic_field_rt<ZMASK>(st[rho], (j0 + 4) * BZ, magic),
                                                            magic_field_rt<ZMASK>(st[rho], (j1 + 4) * BZ, magic)),
                                                make_float2(-kMagic, -kMagic));
                        const float2 shat = fmul2(Ss, fadd2(cs, Zs));
                        const float2 zhat = fmul2(Sz, fadd2(cz, Zz));
                        // integer part of the zero goes into the codes exactly; the
                        // fraction (|.| <= 1/2) is the fp16 addend
                        const float2 zi = make_float2(fminf(fmaxf(rintf(zhat.x), -15.f), 15.f),
                                                      fminf(fmaxf(rintf(zhat.y), -15.f), 15.f));
                        const float2 S0 = fmul2(shat, f0), S1 = fmul2(shat, f1);
                        // 1024 + zi 2^p: exact in binary16 for |zi| <= 15, p <= 7
                        const float2 Z0 = ffma2(zi, g0, make_float2(1024.f, 1024.f));
                        const float2 Z1 = ffma2(zi, g1, make_float2(1024.f, 1024.f));
                        const float2 C = fmul2(fmul2(shat, fadd2(zi, make_float2(-zhat.x, -zhat.y))),
                                               make_float2(sig_scale, sig_scale));
                        const int row = g + 8 * rho;
                        std::uint8_t* te = tab + row * TS + (8 * hi + 2 * t) * 16;
                        *reinterpret_cast<uint4*>(te) =
                            make_uint4(pack_h2_rn(S0.x, S1.x), pack_h2_rn(Z0.x, Z1.x), pack_h2_rn(C.x, 0.f), 0u);
                        *reinterpret_cast<uint4*>(te + 16) =
                            make_uint4(pack_h2_rn(S0.y, S1.y), pack_h2_rn(Z0.y, Z1.y), pack_h2_rn(C.y, 0.f), 0u);
                    }
                }
                __syncwarp();
            }
            // this cell's stages 2it (column half 0) and 2it + 1 (half 1)
            const std::uint32_t ab0 = sb0, an0 = sn0;  // buffer, use count
            const std::uint32_t ab1 = sb0 + 1u == NA ? 0u : sb0 + 1u, an1 = ab1 == 0u ? sn0 + 1u : sn0;
            sb0 += 2u;
            if (sb0 >= NA) {
                sb0 -= NA;
                ++sn0;
            }
            auto do_half = [&](auto HH) {
                constexpr int h_ = decltype(HH)::value;
                const std::uint32_t ab = h_ ? ab1 : ab0;
                std::uint8_t* A = abuf + ab * A_STAGE;
                // only this half's code containers (blocks 8h .. 8h+7), as 8 B loads
                constexpr int W0 = G::CW * (8 * h_ / G::MPC), W1 = G::CW * ((8 * h_ + 7) / G::MPC + 1);
                static_assert(W0 % 2 == 0 && W1 % 2 == 0, "code words of a half: 8 B aligned");
                std::uint32_t cw[G::LANE_WORDS];
#pragma unroll
                for (int i = W0; i < W1; i += 2) {
                    const uint2 w2 = reinterpret_cast<const uint2*>(unit + lane * 16 * BW)[i / 2];
                    cw[i] = w2.x;
                    cw[i + 1] = w2.y;
                }
                const int tb = HPW == 2 ? 8 * h_ : 0;  // this half's first table block
                const std::uint32_t row_sa = smem_u32(A) + (mq >> 1) * KC_A +
                                             (4u * ci + 2u * uu + (mq & 1u)) * 128u + (lane & 7) * 16u;
                // table entries one block ahead of their use (LDS latency)
                uint4 n0 = *reinterpret_cast<const uint4*>(tab + g * TS + tb * 16);
                uint4 n1 = *reinterpret_cast<const uint4*>(tab + (g + 8) * TS + tb * 16);
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                    const int mu = 8 * h_ + jj, cidx = mu / G::MPC, mm = mu % G::MPC;
                    const std::uint32_t* w = cw + G::CW * cidx;
                    const uint4 e0 = n0, e1 = n1;
                    if (jj < 7) {
                        n0 = *reinterpret_cast<const uint4*>(tab + g * TS + (tb + jj + 1) * 16);
                        n1 = *reinterpret_cast<const uint4*>(tab + (g + 8) * TS + (tb + jj + 1) * 16);
                    }
                    std::uint32_t a[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int rho = r & 1, kh = r >> 1, qq = 2 * mm + kh;
                        const int i = rho * (G::NP / 2) + qq;
                        const int Bq = (BW * i) >> 3, pb = (BW * i) & 7;
                        const std::uint32_t code = tc::code_bias<MASK>(window<G::CW>(w, Bq), pb, bias16);
                        const uint4 e = rho ? e1 : e0;
                        a[r] = kh ? tc::deq2<true>(code, e.y, e.x, e.z) : tc::deq2<false>(code, e.y, e.x, e.z);
                    }
                    tc::stsm_x4(row_sa + 2u * jj * KC_A, a[0], a[1], a[2], a[3]);
                }
            };
            // HPW = 2: both halves in one pass, block jj of half 0 next to block jj
            // of half 1 (two independent chains per step for latency hiding)
            auto do_both = [&]() {
                std::uint32_t cw[G::LANE_WORDS];
#pragma unroll
                for (int i = 0; i < G::LANE_WORDS / 4; ++i) {
                    const uint4 w4 = reinterpret_cast<const uint4*>(unit + lane * 16 * BW)[i];
                    cw[4 * i] = w4.x;
                    cw[4 * i + 1] = w4.y;
                    cw[4 * i + 2] = w4.z;
                    cw[4 * i + 3] = w4.w;
                }
                const std::uint32_t rs = (mq >> 1) * KC_A + (4u * ci + 2u * uu + (mq & 1u)) * 128u + (lane & 7) * 16u;
                const std::uint32_t sa[2] = {smem_u32(abuf + ab0 * A_STAGE) + rs, smem_u32(abuf + ab1 * A_STAGE) + rs};
                uint4 n[2][2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    n[h][0] = *reinterpret_cast<const uint4*>(tab + g * TS + (8 * h) * 16);
                    n[h][1] = *reinterpret_cast<const uint4*>(tab + (g + 8) * TS + (8 * h) * 16);
                }
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int mu = 8 * h + jj, cidx = mu / G::MPC, mm = mu % G::MPC;
                        const std::uint32_t* w = cw + G::CW * cidx;
                        const uint4 e0 = n[h][0], e1 = n[h][1];
                        if (jj < 7) {
                            n[h][0] = *reinterpret_cast<const uint4*>(tab + g * TS + (8 * h + jj + 1) * 16);
                            n[h][1] = *reinterpret_cast<const uint4*>(tab + (g + 8) * TS + (8 * h + jj + 1) * 16);
                        }
                        std::uint32_t a[4];
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            const int rho = r & 1, kh = r >> 1, qq = 2 * mm + kh;
                            const int i = rho * (G::NP / 2) + qq;
                            const int Bq = (BW * i) >> 3, pb = (BW * i) & 7;
                            const std::uint32_t code = tc::code_bias<MASK>(window<G::CW>(w, Bq), pb, bias16);
                            const uint4 e = rho ? e1 : e0;
                            a[r] = kh ? tc::deq2<true>(code, e.y, e.x, e.z) : tc::deq2<false>(code, e.y, e.x, e.z);
                        }
                        tc::stsm_x4(sa[h] + 2u * jj * KC_A, a[0], a[1], a[2], a[3]);
                    }
                }
            };
            // this warp's A buffers are free once the MMAs of their previous stages completed
            if (HPW == 2 || h0 == 0)
                if (an0) TC_WAIT(1, mbar_wait(&a_free[ab0], (an0 - 1u) & 1u))
            if (HPW == 2 || h0 == 1)
                if (an1) TC_WAIT(1, mbar_wait(&a_free[ab1], (an1 - 1u) & 1u))
            if (have) {
                if (HPW == 2) {
                    do_both();
                } else if (h0 == 0) {
                    do_half(std::integral_constant<int, 0>{});
                } else {
                    do_half(std::integral_constant<int, 1>{});
                }
            }
            // outliers of the cell: w += v (fp16, scaled by 2^-sigma).  The
            // warps of the cell row own both A buffers of the cell (stages 2it,
            // 2it + 1) between the two row barriers and split the entry list
            // 32 RW ways, so no warp searches for its (unit, half) run
            bar_sync_named(1 + ci, 32 * RW);  // the row's stmatrix writes are done
            if (have) {
                const std::uint32_t cnt = (r1 - r0 - CELL) / 4u;
                const std::uint32_t nfast = (min(r1 - r0, p.rec_cap) - CELL) / 4u;
                const std::uint32_t* es = reinterpret_cast<const std::uint32_t*>(cell + CELL);
                const std::uint32_t* eg = reinterpret_cast<const std::uint32_t*>(p.cells + r0 + CELL);
                const std::uint32_t rowb = (4u * ci) * 128u;
                const std::uint32_t a_h0 = smem_u32(abuf) + ab0 * A_STAGE + rowb;
                const std::uint32_t a_h1 = smem_u32(abuf) + ab1 * A_STAGE + rowb;
#pragma unroll 1
                for (std::uint32_t i = 32u * static_cast<std::uint32_t>(warp >> 2) + lane; i < cnt; i += 32u * RW) {
                    const std::uint32_t e = i < nfast ? es[i] : __ldg(eg + i);
                    const std::uint32_t col = (e >> 16) & 255u, row = e >> 24;
                    if (row < 32u) {
                        const std::uint32_t sa = ((col & 128u) ? a_h1 : a_h0) + ((col & 127u) >> 3) * KC_A +
                                                 (row >> 3) * 128u + (row & 7u) * 16u + (col & 7u) * 2u;
                        unsigned short hb;
                        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(hb) : "r"(sa));
                        const float wv = __half2float(__ushort_as_half(hb)) + h2f_bits(e & 0xffffu) * sig_scale;
                        hb = __half_as_ushort(__float2half_rn(wv));
                        asm volatile("st.shared.u16 [%0], %1;" ::"r"(sa), "h"(hb));
                    }
                }
            }
            fence_proxy_async();               // generic-proxy smem writes -> tensor core reads
            bar_sync_named(1 + ci, 32 * RW);  // ... of every warp of the row
            if (lane == 0) {
                if (HPW == 2 || h0 == 0) mbar_arrive(&a_full[ab0]);
                if (HPW == 2 || h0 == 1) mbar_arrive(&a_full[ab1]);
            }
            if (have) {
                if (lane == 0) mbar_arrive(&rec_empty[ci][sl]);  // this warp is done with the record
                ++k;
            }
            // epilogue after the tile's last unit in this range: the warps of a
            // cell row split the accumulator's 16-column chunks
            const std::uint32_t T_ = tile_of(u), P = u - T_ * p.Pn;
            if (u + 1 == u1 || P + 1 == p.Pn) {
                const std::uint32_t db = tile_i & 1u;
                const std::uint32_t part = static_cast<std::uint32_t>(warp >> 2);  // 0 .. RW-1
                TC_WAIT(2, mbar_wait(&d_full[db], (tile_i >> 1) & 1u))
                tc::fence_after();
                const std::uint32_t row = 128u * T_ + 32u * ci + lane;
                const std::uint32_t ta = tmem + ((32u * ci) << 16) + db * N;
                const std::uint32_t ua = u0 > T_ * p.Pn ? u0 : T_ * p.Pn;  // this range's units of tile T
                const bool whole = ua == T_ * p.Pn && u + 1 == (T_ + 1) * p.Pn;
                const uint2 gm = whole ? make_uint2(0, 0) : __ldg(reinterpret_cast<const uint2*>(p.gmap) + T_);
                const std::uint32_t ord = whole ? 0u : __ldg(p.cmap + 2u * v + (T_ == tile_of(u0) ? 0u : 1u));
                const std::uint32_t Nout = p.Nh ? p.Nh : N;  // output columns of this launch
#pragma unroll 1
                for (std::uint32_t c0 = 16u * part; c0 < Nout; c0 += 16u * RW) {
                    float vv[16];
                    tc::ld16(ta + c0, vv);
                    if (p.Nh) {  // + the lo parts of x
                        float vl[16];
                        tc::ld16(ta + c0 + p.Nh, vl);
#pragma unroll
                        for (int j = 0; j < 16; ++j) vv[j] += vl[j];
                    }
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const std::uint32_t bcol = c0 + j;
                        if (whole) {
                            if (bcol < p.B && row < p.m) p.y[static_cast<std::size_t>(bcol) * p.m + row] = vv[j] * p.out_scale;
                        } else {
                            __stcg(p.partial + (static_cast<std::size_t>(gm.x + ord) * N + bcol) * 128u + 32u * ci + lane,
                                   vv[j]);
                        }
                    }
                }
                tc::fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&d_free[db]);
                if (!whole) {  // last contributor adds the partial tiles in range order
                    std::uint32_t prev = 0;
                    if (lane == 0)
                        asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;"
                                     : "=r"(prev)
                                     : "l"(p.counters + 16u * T_ + warp)
                                     : "memory");
                    prev = __shfl_sync(0xffffffffu, prev, 0);
                    __syncwarp();
                    if (prev == gm.y - 1u) {
#pragma unroll 1
                        for (std::uint32_t c0 = 16u * part; c0 < Nout; c0 += 16u * RW)
                            for (std::uint32_t bcol = c0; bcol < c0 + 16u && bcol < p.B; ++bcol) {
                                float sum = 0.f;
                                for (std::uint32_t j = 0; j < gm.y; ++j)
                                    sum += __ldcg(p.partial + (static_cast<std::size_t>(gm.x + j) * N + bcol) * 128u +
                                                  32u * ci + lane);
                                if (row < p.m) p.y[static_cast<std::size_t>(bcol) * p.m + row] = sum * p.out_scale;
                            }
                        if (lane == 0) p.counters[16u * T_ + warp] = 0;
                    }
                }
                ++tile_i;
            }
        }
    }
#ifdef SPQR_TIMELINE
    if (lane == 0 && blockIdx.x < 148) {
        const std::uint32_t wk = blockIdx.x * 32u + warp;
        g_timeline[8 * wk + 0] = t_start;
        g_timeline[8 * wk + 1] = gtime();
        g_timeline[8 * wk + 2] = tw[0];
        g_timeline[8 * wk + 3] = tw[1];
        g_timeline[8 * wk + 4] = tw[2];
        g_timeline[8 * wk + 5] = u1 - u0;
        g_timeline[8 * wk + 6] = warp;
        g_timeline[8 * wk + 7] = 7;
    }
#endif
    tc::fence_before();
    __syncthreads();
    if (warp == CTRL) {
        tc::fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols));
    }
}
